#!/bin/bash
# ncu launch list of the C5 fine step and a full capture of its interpolation
# (1-row slabs, 16-particle m-units) and warp-owned spread.
mkdir -p gpurun_out
B="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong"
$B > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launches_c4.csv $B > gpurun_out/ncu_list_c4.log 2>&1
echo "list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_interp_push_slab|k_spread_warp" -s 2 -c 2 -o gpurun_out/r2l_full_c4 $B > gpurun_out/ncu_full_c4.log 2>&1
echo "full rc=$?"
