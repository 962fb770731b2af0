#!/bin/bash
# C5-size parareal over the full T = 19.2 (6144 fine steps) on 4 GPUs, PIF coarse
# (run under `gpurun --gpus 4`).
mkdir -p gpurun_out
timeout 2400 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 \
  --master-port 29530 bench_parareal.py --coarse pif --particles 67108864 --T 19.2 \
  > gpurun_out/parareal_c5_T19_4gpu_pif.jsonl 2> gpurun_out/parareal_c5_T19_4gpu_pif.err
true
