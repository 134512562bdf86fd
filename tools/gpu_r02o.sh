#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -s --durations=5 -k "tensor_core or overflow or coherent or determinism or evaluate_host or full_size and cfg3 or sharding and not True" > gpurun_out/pytest_o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_o.log
rm -f gpurun_out/run_cfgs.json
for spec in "3:" "3:" "5:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
timeout 300 python tools/debug/mma_accuracy.py > gpurun_out/mma_acc.txt 2>&1
