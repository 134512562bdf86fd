#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -s -x --durations=5 -k "wide or precondition_gpu or partial or buffer" > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
CMD="python tools/run_cfg.py --config 4 --steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eval_sparse_coop|k_classify" -s 2 -c 2 -o gpurun_out/prof_sparse $CMD > gpurun_out/ncu_sparse.log 2>&1
