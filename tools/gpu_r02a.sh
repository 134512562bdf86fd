#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s --durations=10 -k "confidence or coherent or near_unit or nccl or full_size or overflow" > gpurun_out/pytest_a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_a.log
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-extra > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config 5 --fp32 --steps 5 --warmup 3 --no-extra > gpurun_out/bench_c5f.json 2> gpurun_out/bench_c5f.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-extra --no-e2e > gpurun_out/bench_tr1.json 2> gpurun_out/bench_tr1.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
