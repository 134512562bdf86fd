#!/bin/bash
# Tensor-core phase count (16 vs 32) and CTAs/SM: cfg3 / cfg5 stage times, full-Horner rate, then the
# tensor-core accuracy and determinism tests on the default build.
mkdir -p gpurun_out
rm -f gpurun_out/phases.txt
for F in "" "-DFPE_MMA_PHASES=16" "-DFPE_MMA_MINB=1"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for spec in "3:0" "3:0" "5:0"; do
    cfg=${spec%%:*}; np=${spec#*:}
    echo "[$F] cfg$cfg pts=$np $(python tools/run_cfg.py --config $cfg --points $np --steps 3)" >> gpurun_out/phases.txt
  done
  echo "[$F] horner $(python tools/run_horner.py 1048576)" >> gpurun_out/phases.txt
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -s -k "tensor_core or determinism or coherent or near_unit or horner or full_size and cfg3" > gpurun_out/phases_tests.log 2>&1; echo "rc=$?" >> gpurun_out/phases_tests.log
