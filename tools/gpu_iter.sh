#!/bin/bash
# One iteration: stage times + counters (cfg3 x2, cfg5, cfg5-fp32, cfg2, cfg1), the full-size/sharding/overflow tests, then the GPU suite
mkdir -p gpurun_out
rm -f gpurun_out/iter_times.txt
for spec in "3:" "3:" "5:" "5:--fp32" "2:" "1:"; do
  cfg=${spec%%:*}; extra=${spec#*:}
  timeout 300 python tools/run_cfg.py --config $cfg $extra --steps 3 >> gpurun_out/iter_times.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -s -k "full_size or sharding or overflow or determinism" > gpurun_out/iter_tests.log 2>&1; echo "rc=$?" >> gpurun_out/iter_tests.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/iter_tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/iter_tests_all.log
