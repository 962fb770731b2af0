python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 6 7; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1; done
tail -15 gpurun_out/pytest_gpu.log; for c in 6 7; do python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/bench_c$c.log') if l.startswith('{')][-1]); print($c, d['value'], d['ms_per_step'], d['phase_ms_per_step'])"; done
