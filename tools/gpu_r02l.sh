#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 -k "determinism or tensor_core or overflow or evaluate_host or coherent or wide or cfg1 or near_unit or full_size and cfg3" > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_l.log
rm -f gpurun_out/run_cfgs.json
for spec in "3:" "5:" "5:--fp32" "2:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
for p in 2097152 4194304; do python tools/run_cfg.py --config 3 --points $p --steps 3; done >> gpurun_out/run_cfgs.json 2>&1
timeout 600 python tools/e2e_sweep.py 22:20:6 22:18:6 21:18:8 > gpurun_out/e2e_sweep.txt 2>&1
