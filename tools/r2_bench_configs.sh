#!/bin/bash
# Short bench lines of several configs: CONFIGS="1 6 7" tools/r2_bench_configs.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in ${CONFIGS:-1 6 7}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-strong > gpurun_out/bench_c$c.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c$c.log') if l.startswith('{')][-1]); print($c, '%.4g'%d['value'], '%.3f'%d['ms_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, 'frac %.3f'%d['roofline']['frac'])" || tail -5 gpurun_out/bench_c$c.log
done
