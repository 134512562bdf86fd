#!/bin/bash
# cfg4 (sparse handle): stage times, then one ncu --set full capture of k_eval_sparse_coop + hot lines.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do python tools/run_cfg.py --config 4 --steps 5 >> gpurun_out/sparse_time.txt 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eval_sparse|k_classify" -s 2 -c 2 \
  -o /tmp/prof_sparse python tools/run_cfg.py --config 4 --steps 2 > gpurun_out/ncu_sparse.log 2>&1
python tools/summarize_ncu.py /tmp/prof_sparse.ncu-rep > gpurun_out/ncu_sparse.json 2>&1
python tools/ncu_hotlines.py /tmp/prof_sparse.ncu-rep k_eval_sparse 40 > gpurun_out/ncu_sparse_hot.txt 2>&1
