#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python tools/e2e_sweep.py 22:20:6:0 22:20:6:1 22:21:6:1 22:20:8:1 23:21:4:1 21:19:8:1 > gpurun_out/e2e_sweep.txt 2>&1
timeout 120 python tools/debug/pcie.py > gpurun_out/pcie.txt 2>&1
