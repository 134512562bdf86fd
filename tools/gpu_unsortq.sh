#!/bin/bash
# k_unsort with the per-warp z^l queue: gathers in flight / CTAs per SM variants (cfg3 stage times).
bash tools/gpu_variants_cfg3.sh "" "-DFPE_UNSORT_U=4 -DFPE_UNSORT_MINB=2" "-DFPE_UNSORT_U=3 -DFPE_UNSORT_MINB=2" "-DFPE_UNSORT_MINB=4" "-DFPE_UNSORT_U=1 -DFPE_UNSORT_MINB=4"
mv gpurun_out/var_cfg3.txt gpurun_out/var_unsortq.txt
