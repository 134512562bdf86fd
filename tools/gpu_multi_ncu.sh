#!/bin/bash
# tests + bench + ncu launch list + ncu --set full on several kernels (one capture each, small -c)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_eval_tiled|k_classify_bucket|k_chunk_sort|k_plan|k_bucket_scatter}" -s ${NCU_S:-20} -c ${NCU_C:-5} -o gpurun_out/prof_multi $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/bench.err
