#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eval_tiled" -s 2 -c 1 -o gpurun_out/prof_tiled_small python tools/run_cfg.py --config 3 --points 2097152 --steps 2 > gpurun_out/ncu_small.log 2>&1
bash tools/unsort_variants.sh
