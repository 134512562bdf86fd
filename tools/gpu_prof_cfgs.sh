#!/bin/bash
# Launch lists + one ncu --set full capture of the window evaluator for cfg2 (real) and cfg5-fp32.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "2:" "5:--fp32"; do
  cfg=${spec%%:*}; extra=${spec#*:}; tag=cfg${cfg}${extra:+_fp32}
  CMD="python tools/run_cfg.py --config $cfg $extra --steps 2"
  $CMD > gpurun_out/plain_$tag.json 2> gpurun_out/plain_$tag.err || continue
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches_$tag.csv $CMD > /dev/null 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval_tiled" -s 2 -c 1 \
    -o gpurun_out/prof_eval_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag ncu rc=$?" >> gpurun_out/prof.log
done
