#!/bin/bash
# A/B of library builds on one GPU: AB="cfg:lib1,lib2 cfg:lib3" tools/r2_ab.sh
mkdir -p gpurun_out
for spec in $AB; do
  c=${spec%%:*}; libs=${spec#*:}
  for lib in ${libs//,/ }; do
    PIF_LIBRARY=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong > gpurun_out/ab.log 2>&1
    python -c "
import json
try:
    d=json.loads([l for l in open('gpurun_out/ab.log') if l.startswith('{')][-1]); print('cfg $c', '$lib', '%.4g'%d['value'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, 'frac %.3f'%d['roofline']['frac'])
except Exception as e: print('cfg $c', '$lib', 'FAILED', open('gpurun_out/ab.log').read()[-800:])
"
  done
done
true
