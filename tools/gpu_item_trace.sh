#!/bin/bash
# k_eval_tiled per-item timeline at small batches (debug build), then the normal build back.
mkdir -p gpurun_out
FPE_EXTRA_FLAGS="-DFPE_ITEM_TRACE" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
for n in ${TRACE_N:-1048576 2097152}; do python tools/item_trace.py $n >> gpurun_out/item_trace.txt 2>&1; done
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
