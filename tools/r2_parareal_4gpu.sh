#!/bin/bash
# C5-size parareal on 4 GPUs (gpurun --gpus 4): Landau, 64^3 modes, 2^26
# particles, T = 2.4, fine eps 1e-7 / dt 0.003125, coarse dt_g = 0.05; speedups
# vs serial fine (1 GPU) and vs the particle-decomposed fine on all 4 GPUs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
run() {  # name, args
  timeout 1200 $TR --master-port $((29600 + RANDOM % 300)) bench_parareal.py --particles 67108864 "${@:2}" \
    > gpurun_out/r2_parareal_$1.jsonl 2> gpurun_out/r2_parareal_$1.err
  echo "$1 rc=$?"; tail -c 1500 gpurun_out/r2_parareal_$1.jsonl
}
run t4_pif32 --coarse pif32
run t4_pif --coarse pif --no-space-ref
run t4_pic --coarse pic --no-space-ref
run s2t2_pif32 --coarse pif32 --space 2 --no-space-ref
true
