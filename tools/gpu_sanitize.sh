#!/bin/bash
# memcheck on small parity tests (one sanitizer tool per call), then a torchrun N=1 bench (NCCL path)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "cfg1_all_points or empty_and_ragged or special_points or worked_example or buffer_roundtrip or horner" \
  > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err
echo "torchrun rc=$?" >> gpurun_out/torchrun1.err
