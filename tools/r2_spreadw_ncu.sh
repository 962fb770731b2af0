#!/bin/bash
# Full ncu captures of the warp-owned spread (C5 fine w = 8, C5 coarse fp32 w = 5).
mkdir -p gpurun_out
for c in 4 8; do
  ncu --set full --clock-control none --import-source on -k regex:"k_spread_warp|k_bin_count" -s 2 -c 2 -o gpurun_out/r2g_full_c$c \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong > gpurun_out/ncu_full_c$c.log 2>&1
  echo "full c$c rc=$?"
done
ls -la gpurun_out/r2g_full_c*.ncu-rep
