#!/bin/bash
# ncu --set full of k_eval_tiled for one experiment build (VARIANT), after a plain run of the same command
mkdir -p gpurun_out
cp paper_2211_06320_b200/libfpe_${VARIANT}.so paper_2211_06320_b200/libfpe.so
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra"
$CMD > gpurun_out/plain_var.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_tiled -s 2 -c 1 -o gpurun_out/prof_${VARIANT} $CMD > gpurun_out/ncu_var.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_var.log
