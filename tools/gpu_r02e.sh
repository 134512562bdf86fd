#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -x --durations=5 -k "dtype or coherent or near_unit or cfg5_fp32 or determinism or evaluate_host or horner or special_points_fp32 or wide" > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e.log
for spec in "5:--fp32" "2:" "3:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
CMD="python tools/run_cfg.py --config 3 --steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eval_tiled" -s 2 -c 1 -o gpurun_out/prof_tiled_cfg3 $CMD > gpurun_out/ncu_tiled.log 2>&1
