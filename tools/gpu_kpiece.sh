#!/bin/bash
# kPiece (the absolute piece length of long windows / the tensor-core item) variants: cfg3 full and 2^21-point
# batches, cfg5; then the tensor-core / determinism tests on the default build.
mkdir -p gpurun_out
rm -f gpurun_out/kpiece.txt
for F in "" "-DFPE_KPIECE=8192" "-DFPE_KPIECE=4096"; do
  FPE_EXTRA_FLAGS="$F" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
  for spec in "3:0" "3:0" "3:2097152" "3:1048576" "5:0"; do
    cfg=${spec%%:*}; np=${spec#*:}
    echo "[$F] cfg$cfg pts=$np $(python tools/run_cfg.py --config $cfg --points $np --steps 3)" >> gpurun_out/kpiece.txt
  done
done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "tensor_core or determinism or coherent or near_unit or full_size and cfg3" > gpurun_out/kpiece_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kpiece_tests.log
