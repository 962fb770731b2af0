#!/bin/bash
# Round-2 single-GPU measurement batch: GPU suite, smoke, bench lines (C2
# default with e2e / cpu_baseline / c3_strong, other configs short), reference
# arm, convergence slopes, then the ncu launch list and full captures.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.jsonl 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
for c in 2 3 4 7 8 10; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c$c.jsonl 2> gpurun_out/r2_bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.jsonl 2>&1; echo "ref rc=$?"
for m in eps dtg pc h; do
  timeout 1500 python tools/slopes.py $m > gpurun_out/r2_slopes_$m.json 2> gpurun_out/r2_slopes_$m.err; echo "slopes $m rc=$?"
done
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-c3-strong"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $B > gpurun_out/ncu_list.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_interp_push_slab|k_spread|k_bin_count|k_gather_sorted|k_scatter_index" -s 10 -c 5 -o gpurun_out/r2_full $B > gpurun_out/ncu_full.log 2>&1
B7="python bench.py --config 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c3-strong"
$B7 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_interp_push_simt|k_spread" -s 2 -c 2 -o gpurun_out/r2_full_c8 $B7 > gpurun_out/ncu_full_c8.log 2>&1
echo "ncu rc=$?"; ls gpurun_out/*.ncu-rep
true
