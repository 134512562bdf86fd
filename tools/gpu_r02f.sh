#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 -k "cfg1 or special or dtype or sparse or ragged or newton or horner_context or evaluate_host or half_circle or second_point" > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.log
timeout 900 python tools/e2e_sweep.py 22:18:6 22:16:6 22:20:6 22:21:6 22:18:8 21:17:8 > gpurun_out/e2e_sweep.txt 2>&1
FPE_HOST_TRACE=1 timeout 300 python tools/debug/e2e_trace.py > gpurun_out/e2e_trace.txt 2>&1
for spec in "3:" "5:--fp32" "2:" "1:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/run_cfgs.json 2>&1
done
