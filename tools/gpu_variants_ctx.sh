#!/bin/bash
# A/B of experiment builds including the bench's context configs (cfg1/2/4/5/5_fp32)
mkdir -p gpurun_out
cp paper_2211_06320_b200/libfpe.so /tmp/libfpe_base.so
for V in base ${VARIANTS}; do
  if [ "$V" != base ]; then cp paper_2211_06320_b200/libfpe_$V.so paper_2211_06320_b200/libfpe.so; else cp /tmp/libfpe_base.so paper_2211_06320_b200/libfpe.so; fi
  timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 10 ${BENCH_ARGS} > gpurun_out/varc_$V.json 2> gpurun_out/varc_$V.err
done
cp /tmp/libfpe_base.so paper_2211_06320_b200/libfpe.so
