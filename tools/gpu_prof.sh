#!/bin/bash
# ncu launch list + full captures of the evaluator and the radix downsweep
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
CMD2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --points 8388608"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_eval_tiled|k_radix_downsweep|k_classify_sort" -s 0 -c 5 -o gpurun_out/prof_tiled $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
