#!/bin/bash
# k_bucket_scatter variants (loads in flight, CTAs per SM): cfg3 stage times.
bash tools/gpu_variants_cfg3.sh "" "-DFPE_SCATTER_U=8" "-DFPE_SCATTER_MINB=8" "-DFPE_SCATTER_U=8 -DFPE_SCATTER_MINB=6" "-DFPE_SCATTER_U=2 -DFPE_SCATTER_MINB=8"
mv gpurun_out/var_cfg3.txt gpurun_out/var_scatter.txt
