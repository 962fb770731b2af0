#!/bin/bash
# Round-2 closing 4-GPU batch (gpurun --gpus 4), after the fused sort: the whole
# GPU suite (multi-GPU tests vs the oracle included), bench at N = 1 / 2 / 4
# (self-spawned ranks), C5-size parareal (PIF fp32 coarse, space-only reference).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2i_pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2i_pytest_gpu_4gpu.log
for N in 1 2 4; do
  timeout 600 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2i_bench_n$N.jsonl 2> gpurun_out/r2i_bench_n$N.err
  echo "bench N=$N rc=$?"; tail -c 300 gpurun_out/r2i_bench_n$N.jsonl
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
run() {  # name, args
  timeout 1500 $TR --master-port $((29600 + RANDOM % 300)) bench_parareal.py "${@:2}" \
    > gpurun_out/r2i_parareal_$1.jsonl 2> gpurun_out/r2i_parareal_$1.err
  echo "$1 rc=$?"; grep '^{' gpurun_out/r2i_parareal_$1.jsonl | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print({k: d.get(k) for k in ['value','speedup_vs_space_only','space_only_speedup_vs_serial','t_serial_s','t_space_only_s','t_parareal_s','iterations','retired_at']})"
}
run p26_t4_pif32 --particles 67108864 --coarse pif32
run p26_s2t2_pif32 --particles 67108864 --coarse pif32 --space 2 --no-space-ref
true
