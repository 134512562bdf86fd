#!/bin/bash
# first GPU measurement round: bench + ncu launch list + ncu full capture of the top kernel
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --points 4194304"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_eval $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
