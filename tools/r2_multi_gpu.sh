#!/bin/bash
# Round-2 4-GPU batch (gpurun --gpus 4): multi-GPU tests (vs the oracle), the
# self-spawned bench at N = 2 / 4, and C5-size parareal (space x time).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/r2_pytest_multi.log 2>&1; echo "multi rc=$?"; tail -3 gpurun_out/r2_pytest_multi.log
for N in 2 4; do
  timeout 600 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2_bench_n$N.jsonl 2> gpurun_out/r2_bench_n$N.err
  echo "bench N=$N rc=$?"; grep -c "nRanks $N" gpurun_out/r2_bench_n$N.err; tail -c 600 gpurun_out/r2_bench_n$N.jsonl
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
run() {  # name, args
  timeout 1500 $TR --master-port $((29600 + RANDOM % 300)) bench_parareal.py --particles 67108864 "${@:2}" \
    > gpurun_out/r2_parareal_$1.jsonl 2> gpurun_out/r2_parareal_$1.err
  echo "$1 rc=$?"; tail -c 400 gpurun_out/r2_parareal_$1.jsonl
}
run t4_pif32 --coarse pif32
run t4_pif --coarse pif --no-space-ref
run t4_pic --coarse pic --no-space-ref
run s2t2_pif32 --coarse pif32 --space 2 --no-space-ref
run s2t2_pic --coarse pic --space 2 --no-space-ref
true
