#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/np_variants.txt
for np in 4 8; do
  FPE_EXTRA_FLAGS="-DFPE_NP_F32=$np" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  echo "NP_F32=$np $(python tools/run_cfg.py --config 5 --fp32 --steps 3)" >> gpurun_out/np_variants.txt
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
