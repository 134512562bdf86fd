#!/bin/bash
# cfg3 stage times under experiment flags given as arguments ("" = the default build).
mkdir -p gpurun_out
rm -f gpurun_out/var_cfg3.txt
for F in "$@"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for i in 1 2; do echo "[$F] $(python tools/run_cfg.py --config ${CFG:-3} --steps 3)" >> gpurun_out/var_cfg3.txt; done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
