#!/bin/bash
# Round-2 closing 4-GPU parareal batch (final kernels):
# parareal vs space-only at 2^22 and 2^26 (C5), PIF fp32 / fp64 and CIC-PIC
# coarse, space x time 2 x 2.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
run() {  # name, args
  timeout 1500 $TR --master-port $((29600 + RANDOM % 300)) bench_parareal.py "${@:2}" \
    > gpurun_out/r2j_parareal_$1.jsonl 2> gpurun_out/r2j_parareal_$1.err
  echo "$1 rc=$?"; grep '^{' gpurun_out/r2j_parareal_$1.jsonl | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print({k: d.get(k) for k in ['value','speedup_vs_space_only','space_only_speedup_vs_serial','t_serial_s','t_space_only_s','t_parareal_s','iterations','retired_at']})"
}
run p26_t4_pif32 --particles 67108864 --coarse pif32
run p26_s2t2_pif32 --particles 67108864 --coarse pif32 --space 2 --no-space-ref
run p26_t4_pif --particles 67108864 --coarse pif --no-space-ref
run p26_t4_pic --particles 67108864 --coarse pic --no-space-ref
true
