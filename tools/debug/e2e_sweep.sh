#!/bin/bash
# e2e (host buffers) timing of fpe_evaluate_host for several pipeline settings: "chunk:first:slots"
mkdir -p gpurun_out
for S in ${SETTINGS:-23:22:4}; do
  IFS=: read C F N <<< "$S"
  FPE_HOST_CHUNK_LOG2=$C FPE_HOST_FIRST_LOG2=$F FPE_HOST_SLOTS=$N timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 3 --e2e-steps 5 > gpurun_out/e2e_$C_$F_$N.json 2>/dev/null
  python -c "import json;b=json.loads(open('gpurun_out/e2e_$C_$F_$N.json').read().strip().splitlines()[-1]);print('$S', round(b['e2e']['ms_per_step'],2))" >> gpurun_out/e2e_sweep.txt
done
