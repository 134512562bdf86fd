#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/np_real.txt
for np in 4 2 8; do
  FPE_EXTRA_FLAGS="-DFPE_NP_REAL=$np" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for i in 1 2 3; do echo "NP_REAL=$np $(python tools/run_cfg.py --config 2 --steps 5)" >> gpurun_out/np_real.txt; done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
