#!/bin/bash
# Round-2 closing measurements on one GPU after the fused sort (A/B of the 1-row slab warp count first):
# reference arm, ncu launch list + full capture of the C2 step kernels.
mkdir -p gpurun_out
AB="4:build_ab/libpif_nw24.so,build_ab/libpif_nw16.so,build_ab/libpif_nw20.so,build_ab/libpif_nw24.so,build_ab/libpif_nw16.so" bash tools/r2_ab.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2i_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.jsonl 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
for c in 2 3 4 7 8 10 11; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-c3-strong > gpurun_out/r2i_bench_c$c.jsonl 2> gpurun_out/r2i_bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2i_bench_reference.jsonl 2>&1; echo "ref rc=$?"
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-c3-strong"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv $B > gpurun_out/ncu_list.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_interp_push_slab|k_spread|k_bin_count|k_gather_sorted|k_scatter_index" -s 10 -c 5 -o gpurun_out/r2i_full $B > gpurun_out/ncu_full.log 2>&1
B10="python bench.py --config 10 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c3-strong"
$B10 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_cic|k_pic" -s 3 -c 3 -o gpurun_out/r2i_full_c10 $B10 > gpurun_out/ncu_full_c10.log 2>&1
echo "ncu rc=$?"; ls gpurun_out/r2f*.ncu-rep
true
