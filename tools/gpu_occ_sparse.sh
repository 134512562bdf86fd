#!/bin/bash
# cfg4 sparse evaluator: occupancy / scheduler / per-SM activity spread (ncu), to locate idle SM time.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats --section SpeedOfLight \
  --metrics sm__cycles_active.min,sm__cycles_active.max,sm__cycles_active.avg,smsp__cycles_active.min,smsp__cycles_active.max,sm__warps_active.min,sm__warps_active.max,smsp__warps_launched.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:"k_eval_sparse" -s 1 -c 1 python tools/run_cfg.py --config 4 --steps 1 > gpurun_out/occ_sparse.txt 2>&1
