#!/bin/bash
# staged-accumulator layout experiment: stage times on cfg3 / cfg5 / cfg5-fp32 / cfg2 / cfg4, then the GPU suite
mkdir -p gpurun_out
rm -f gpurun_out/w_times.txt
for spec in "3:" "3:" "5:" "5:--fp32" "2:" "4:" "1:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/w_times.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w_tests.log
