#!/bin/bash
# Round-2 4-GPU batch 2: self-spawned bench at N = 2 / 4 (no torchrun), C5-size
# parareal with fp32 PIF coarse against serial and space-only fine.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for N in 1 2 4; do
  timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2b_bench_n$N.jsonl 2> gpurun_out/r2b_bench_n$N.err
  echo "bench N=$N rc=$?"; tail -c 300 gpurun_out/r2b_bench_n$N.jsonl
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 1500 $TR --master-port 29711 bench_parareal.py --particles 67108864 --coarse pif32 \
  > gpurun_out/r2b_parareal_t4_pif32.jsonl 2> gpurun_out/r2b_parareal_t4_pif32.err
echo "parareal rc=$?"; tail -c 600 gpurun_out/r2b_parareal_t4_pif32.jsonl
true
