#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 -k "determinism or tensor_core or dtype or ragged or coherent or many_vertex or wide" > gpurun_out/pytest_m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_m.log
rm -f gpurun_out/run_cfgs.json
for spec in "3:" "5:" "5:--fp32" "2:" "2:" "2:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
for p in 2097152 4194304; do python tools/run_cfg.py --config 3 --points $p --steps 3; done >> gpurun_out/run_cfgs.json 2>&1
FPE_EXTRA_FLAGS=-DFPE_ITEM_TRACE python -m paper_2211_06320_b200.build --force > gpurun_out/build_tr.log 2>&1
python tools/item_trace.py 2097152 > gpurun_out/trace21.txt 2>&1
python tools/item_trace.py 67108864 > gpurun_out/trace26.txt 2>&1
