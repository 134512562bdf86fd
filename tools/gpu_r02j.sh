#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 -k "horner or sparse or cfg4 or wide" > gpurun_out/pytest_j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_j.log
python tools/run_horner.py 1048576 > gpurun_out/horner.json 2>&1
python tools/run_horner.py 131072 >> gpurun_out/horner.json 2>&1
timeout 300 python tools/run_cfg.py --config 4 --steps 3 > gpurun_out/run_cfg4.json 2>&1
