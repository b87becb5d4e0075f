python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for args in "" "--flush-period 8" "--flush-period 16" "--flush-period 32" "--history-bits 128 --flush-period 32" "--history-bits 128 --flush-period 64"; do
timeout 300 python bench.py --steps 3200 --warmup 320 --no-cpu-baseline --no-e2e $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$args', 'ms/step', round(d['ms_per_step']*1e3,2), {k: round(v*1e3,2) for k,v in d['roofline']['phase_ms_per_step'].items() if k in ('FRONT','STDP','DELIVERY')}, 'flush/step', round(d['per_step']['flush_rows']), 'syn/step', round(d['per_step']['stdp_syn']))"
done
SNN_TRACE_KW='{"flush_period": 16}' SNN_TRACE_T0=1501 timeout 300 python scripts/trace.py 3 0 2>&1 | grep "^stdp"
