#!/bin/bash
# cfg4 sparse evaluator: build-flag variants (long-list threshold, min CTAs per SM), stage times; chunk trace.
mkdir -p gpurun_out
rm -f gpurun_out/sparse_var.txt
for F in "-DFPE_SP_MINB=4" "-DFPE_SP_MINB=4 -DFPE_SP_LONG=32" "-DFPE_SP_MINB=5 -DFPE_SP_LONG=32" "-DFPE_SP_MINB=4 -DFPE_SP_LONG=64"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  grep -A3 "sparse_coopILi1ELi1ELi1" paper_2211_06320_b200/_build/kernels.cu.o.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' ' >> gpurun_out/sparse_var.txt
  for i in 1 2; do echo "[$F] $(python tools/run_cfg.py --config 4 --steps 5)" >> gpurun_out/sparse_var.txt; done
done
FPE_EXTRA_FLAGS="-DFPE_ITEM_TRACE -DFPE_SP_MINB=4" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
python tools/sp_trace.py > gpurun_out/sp_trace.txt 2>&1
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "sparse or cfg4 or determinism" > gpurun_out/sparse_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sparse_tests.log
