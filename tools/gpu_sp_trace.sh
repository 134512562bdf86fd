#!/bin/bash
# cfg4 sparse evaluator: per-chunk timeline (debug build), then the normal build back.
mkdir -p gpurun_out
FPE_EXTRA_FLAGS="-DFPE_ITEM_TRACE" python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
python tools/sp_trace.py > gpurun_out/sp_trace.txt 2>&1
python -m paper_2211_06320_b200.build --force > /dev/null 2>&1
