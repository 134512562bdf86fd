#!/bin/bash
# k_unsort variants (gathers in flight x CTAs/SM register budget): cfg3 stage times
mkdir -p gpurun_out
for v in "4:1" "2:1" "2:2" "4:2" "1:3" "2:3"; do
  U=${v%%:*}; B=${v#*:}
  FPE_EXTRA_FLAGS="-DFPE_UNSORT_U=$U -DFPE_UNSORT_MINB=$B" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  echo "U=$U MINB=$B $(python tools/run_cfg.py --config 3 --steps 3)" >> gpurun_out/unsort_variants.txt
  grep -A2 "k_unsortILi1ELi1" paper_2211_06320_b200/_build/eval_tiled.cu.o.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' ' >> gpurun_out/unsort_variants.txt; echo >> gpurun_out/unsort_variants.txt
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
