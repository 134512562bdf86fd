#!/bin/bash
# A/B timing of experiment builds (libfpe_<V>.so shipped in-tree): bench line per variant
mkdir -p gpurun_out
cp paper_2211_06320_b200/libfpe.so /tmp/libfpe_base.so
for V in base ${VARIANTS}; do
  if [ "$V" != base ]; then cp paper_2211_06320_b200/libfpe_$V.so paper_2211_06320_b200/libfpe.so; else cp /tmp/libfpe_base.so paper_2211_06320_b200/libfpe.so; fi
  timeout 300 python bench.py --no-extra --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/var_$V.json 2> gpurun_out/var_$V.err
done
cp /tmp/libfpe_base.so paper_2211_06320_b200/libfpe.so
