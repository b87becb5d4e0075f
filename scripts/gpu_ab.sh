python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for env in "SNN_X=1" "SNN_X=2"; do
env $env timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$env', 'ms/step', round(d['ms_per_step']*1e3,2), {k: round(v*1e3,2) for k,v in d['roofline']['phase_ms_per_step'].items() if k in ('FRONT','STDP','DELIVERY')})"
done
