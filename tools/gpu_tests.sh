#!/bin/bash
# GPU test suite + a short bench (plain, no ncu)
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -i "model name\|^CPU(s)" >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -s ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
