#!/bin/bash
# stage times of cfg3 (x2), cfg5, cfg5-fp32 under experiment flags given as arguments ("" = the default build)
mkdir -p gpurun_out
rm -f gpurun_out/var2.txt
for F in "$@"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for spec in ${SPECS:-"3:" "3:" "5:" "5:--fp32" "2:"}; do
    cfg=${spec%%:*}; extra=${spec#*:}
    echo "[$F] $(timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 2>&1 | tail -1)" >> gpurun_out/var2.txt
  done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
