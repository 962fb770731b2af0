#!/bin/bash
# A/B the step phases of several libpif builds on one GPU: [AB_ARGS="--config 5"] tools/ab_bench.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for lib in "$@"; do
  PIF_LIBRARY=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong $AB_ARGS > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$lib', round(d['value']/1e6,1), 'Mp/s', {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
except Exception as e: print('$lib', 'FAILED')
"
  grep -m2 -i error gpurun_out/ab.log
done
