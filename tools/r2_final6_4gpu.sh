#!/bin/bash
# Closing check after the 16-particle m-units (gpurun --gpus 4): whole GPU suite,
# C5 fine bench lines on GPU 0, C5-size parareal (PIF fp32 coarse, space-only ref).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2l_pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2l_pytest_gpu_4gpu.log
export CUDA_VISIBLE_DEVICES=0
for c in 4 11; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-c3-strong > gpurun_out/r2l_bench_c$c.jsonl 2> gpurun_out/r2l_bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench.jsonl 2> gpurun_out/r2l_bench.err; echo "bench rc=$?"
unset CUDA_VISIBLE_DEVICES
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 1500 $TR --master-port $((29600 + RANDOM % 300)) bench_parareal.py --particles 67108864 --coarse pif32 \
  > gpurun_out/r2l_parareal_p26_t4_pif32.jsonl 2> gpurun_out/r2l_parareal_p26_t4_pif32.err; echo "parareal rc=$?"
true
