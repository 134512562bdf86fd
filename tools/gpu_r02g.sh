#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
rm -f gpurun_out/run_cfgs.json
for spec in "3:" "5:--fp32" "5:" "2:" "1:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
