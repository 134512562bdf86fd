#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/np_more.txt
for v in "-DFPE_NP_REAL=1:2" "-DFPE_NP_F32=2:5 --fp32" "-DFPE_NP_F32=4:5 --fp32"; do
  F=${v%%:*}; C=${v#*:}
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for i in 1 2; do echo "$F $(python tools/run_cfg.py --config $C --steps 3)" >> gpurun_out/np_more.txt; done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
