#!/bin/bash
# fused-exchange checks on one GPU: the multi-process IPC test, then the bench
# through torchrun (N=1, the fused path with one target) vs plain python
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/fused_tests.log 2>&1
echo "fused tests rc=$?"
tail -5 gpurun_out/fused_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
  > gpurun_out/fused_bench_torchrun.log 2>&1
echo "torchrun fused rc=$?"
tail -1 gpurun_out/fused_bench_torchrun.log | cut -c1-600
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --exchange nccl \
  > gpurun_out/nccl_bench_torchrun.log 2>&1
echo "torchrun nccl rc=$?"
tail -1 gpurun_out/nccl_bench_torchrun.log | cut -c1-600
