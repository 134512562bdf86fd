#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ev_variants.txt
for F in "-DFPE_EVAL_MIN_CTAS=3" "-DFPE_EVAL_MIN_CTAS=4" "-DFPE_MMA_STAGES=6" "-DFPE_MMA_STAGES=3"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  grep -A2 "k_eval_tiledILi1ELi1ELi1ELi4" paper_2211_06320_b200/_build/eval_tiled.cu.o.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' ' >> gpurun_out/ev_variants.txt
  for i in 1 2; do echo "$F | $(python tools/run_cfg.py --config 3 --steps 3)" >> gpurun_out/ev_variants.txt; done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
