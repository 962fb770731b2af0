set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1d_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/r1d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1d_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r1d_smoke.log
timeout 400 python bench.py > gpurun_out/r1d_bench.jsonl 2> gpurun_out/r1d_bench.err
timeout 400 python bench.py --config 2 > gpurun_out/r1d_bench_c3.jsonl 2>> gpurun_out/r1d_bench.err
timeout 400 python bench.py --config 3 > gpurun_out/r1d_bench_c4.jsonl 2>> gpurun_out/r1d_bench.err
timeout 400 python bench.py --config 4 > gpurun_out/r1d_bench_c5f.jsonl 2>> gpurun_out/r1d_bench.err
timeout 400 python bench.py --config 7 > gpurun_out/r1d_bench_c5c.jsonl 2>> gpurun_out/r1d_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1d_bench_ref.jsonl 2>> gpurun_out/r1d_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1d_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1d_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_interp_push|k_spread|k_gather|k_scatter|k_bin" -s 10 -c 5 -o gpurun_out/r1d_full python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1d_ncu_full.log 2>&1
ls -la gpurun_out
