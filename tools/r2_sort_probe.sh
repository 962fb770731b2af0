#!/bin/bash
# Launch lists of the C5 coarse (fp32) and fine steps (sort kernel breakdown) and
# a full capture of the warp-owned spread at C5 fine.
mkdir -p gpurun_out
for c in 8 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_c$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong > gpurun_out/ncu_list_c$c.log 2>&1
  echo "list c$c rc=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"k_spread_warp" -s 4 -c 2 -o gpurun_out/r2g_full_c4 \
  python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong > gpurun_out/ncu_full_c4.log 2>&1
echo "full rc=$?"
