#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 -k "sparse or cfg4 or buffer_roundtrip or wide" > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p.log
rm -f gpurun_out/run_cfgs.json
for i in 1 2; do timeout 300 python tools/run_cfg.py --config 4 --steps 3 >> gpurun_out/run_cfgs.json 2>&1; done
