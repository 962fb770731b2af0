#!/bin/bash
# Round-2 closing measurements (gpurun --gpus 4): the whole GPU suite (multi-GPU
# tests included), smoke, bench default line + --gpus 2 / 4 (self-spawned
# ranks), the --config lines on one GPU, the reference arm, the ncu launch list
# and --set full capture of the default (C2) step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2j_pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2j_pytest_gpu_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo "smoke rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench.jsonl 2> gpurun_out/r2j_bench.err; echo "bench rc=$?"
for c in 2 3 4 7 8 10 11; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-c3-strong > gpurun_out/r2j_bench_c$c.jsonl 2> gpurun_out/r2j_bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2j_bench_reference.jsonl 2>&1; echo "ref rc=$?"
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-c3-strong"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches.csv $B > gpurun_out/ncu_list.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_interp_push_slab|k_spread|k_bin_count|k_scatter_index" -s 8 -c 4 -o gpurun_out/r2j_full $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
unset CUDA_VISIBLE_DEVICES
for N in 2 4; do
  timeout 600 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2j_bench_n$N.jsonl 2> gpurun_out/r2j_bench_n$N.err
  echo "bench N=$N rc=$?"
done
ls gpurun_out/r2j*
true
