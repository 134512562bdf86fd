#!/bin/bash
# unsort register-budget variants (cfg3 / cfg5 / cfg5-fp32 stage times), then the GPU suite on the default build
mkdir -p gpurun_out
bash tools/gpu_variants2.sh "" "-DFPE_UNSORT_MINB=4" "-DFPE_UNSORT_U=1 -DFPE_UNSORT_MINB=4" "-DFPE_UNSORT_U=4 -DFPE_UNSORT_MINB=2"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/y_tests.log
grep -h "counters" gpurun_out/y_tests.log | head -3
