#!/bin/bash
# fpe_evaluate_host: per-chunk timeline (FPE_HOST_TRACE) and a pipeline-setting sweep, cfg3 2^26 points.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
FPE_HOST_TRACE=1 python tools/debug/e2e_trace.py > gpurun_out/e2e_trace.txt 2>&1
python tools/e2e_sweep.py 22:20:6 22:16:6 22:17:6 23:18:6 22:20:4 > gpurun_out/e2e_sweep.txt 2>&1
