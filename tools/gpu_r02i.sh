#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/run_horner.py > gpurun_out/horner.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_horner_tiled" -s 2 -c 1 -o gpurun_out/prof_horner python tools/run_horner.py 32768 > gpurun_out/ncu_horner.log 2>&1
