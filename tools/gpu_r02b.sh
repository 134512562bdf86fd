#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -x --durations=5 -k "sparse or cfg4 or special or ragged or dtype" > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 300 python tools/run_cfg.py --config 4 --steps 3 > gpurun_out/run_cfg4.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
