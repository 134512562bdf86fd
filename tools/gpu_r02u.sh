#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/np_c64.txt
for F in "-DFPE_NO_MMA_ITEMS=1" "-DFPE_NO_MMA_ITEMS=1 -DFPE_NP_C64_LONG=2"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for i in 1 2; do echo "$F | $(python tools/run_cfg.py --config 3 --steps 3)" >> gpurun_out/np_c64.txt; done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
