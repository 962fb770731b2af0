#!/bin/bash
# C5-size parareal on 4 GPUs (run under `gpurun --gpus 4`): Landau, 64^3 modes,
# 2^26 particles (32 per upsampled cell: the dense slab tiles), T = 2.4,
# 4 time slices, coarse = PIF eps 1e-4 or CIC-PIC 32^3, both at dt_g = 0.05.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for G in pif pic; do
  timeout 1500 $TR --master-port 29520 bench_parareal.py --coarse $G --particles 67108864 \
    > gpurun_out/parareal_c5_4gpu_$G.jsonl 2> gpurun_out/parareal_c5_4gpu_$G.err
done
true
