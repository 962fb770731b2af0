#!/bin/bash
# Multi-GPU measurement batch (run under `gpurun --gpus 4`): GPU test suite on 4
# GPUs, bench.py weak-scaling lines at N = 2 and 4, parareal speedup at 4 GPUs.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
for N in 2 4; do
  timeout 600 $TR --nproc-per-node $N --master-port $((29500 + N)) bench.py --gpus $N \
    > gpurun_out/bench_n$N.jsonl 2> gpurun_out/bench_n$N.err
done
for G in pif pic; do
  timeout 900 $TR --nproc-per-node 4 --master-port 29510 bench_parareal.py --coarse $G \
    > gpurun_out/parareal_4gpu_$G.jsonl 2> gpurun_out/parareal_4gpu_$G.err
done
true
