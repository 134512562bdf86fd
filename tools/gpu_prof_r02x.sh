#!/bin/bash
# ncu --set full of every kernel of one cfg3 step (after the same command exits 0 without ncu), summaries on the box
mkdir -p gpurun_out
C3="python tools/run_cfg.py --config 3 --steps 1"
$C3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 8 -c 8 -o /tmp/prof_cfg3_x $C3 > gpurun_out/ncu_cfg3_x.log 2>&1
python tools/summarize_ncu.py /tmp/prof_cfg3_x.ncu-rep > gpurun_out/r02x_ncu_cfg3_all_kernels.json
rm -f gpurun_out/r02x_ncu_cfg3_hotlines.txt
for k in k_classify_bucket k_bucket_hist k_plan k_unsort k_eval_tiled; do python tools/ncu_hotlines.py /tmp/prof_cfg3_x.ncu-rep $k 25 >> gpurun_out/r02x_ncu_cfg3_hotlines.txt; done
cp /tmp/prof_cfg3_x.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
