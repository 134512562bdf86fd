#!/bin/bash
# ncu --set full of one kernel at the bench's full size (plain run first, then ncu on the same command)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
$CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_eval_tiled}" -s ${NCU_S:-4} -c 1 -o gpurun_out/${NCU_OUT:-prof_full} $CMD > gpurun_out/ncu_full2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full2.log
