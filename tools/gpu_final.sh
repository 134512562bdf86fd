#!/bin/bash
# The driver's round-end sequence: GPU tests, smoke, bench (N=1), reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s --durations=15 > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?" >> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config 5 --fp32 --steps 5 --warmup 3 --no-extra > gpurun_out/bench_c5f.json 2> gpurun_out/bench_c5f.err
