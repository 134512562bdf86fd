#!/bin/bash
# cfg3: one ncu --set full capture of the non-evaluator kernels (classify, scatter, plan, unsort) + hot lines.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_classify_bucket|k_bucket_scatter|k_unsort|k_plan" -s 4 -c 4 \
  -o /tmp/prof_aux python tools/run_cfg.py --config 3 --steps 2 > gpurun_out/ncu_aux.log 2>&1
python tools/summarize_ncu.py /tmp/prof_aux.ncu-rep > gpurun_out/ncu_aux.json 2>&1
for k in k_classify_bucket k_bucket_scatter k_unsort k_plan; do
  python tools/ncu_hotlines.py /tmp/prof_aux.ncu-rep $k 30 > gpurun_out/ncu_aux_hot_$k.txt 2>&1
done
