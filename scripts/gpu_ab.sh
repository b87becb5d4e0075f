python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for env in "SNN_X=1" "SNN_STDP_NO_TABLE=1"; do
env $env timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$env ms/step', d['ms_per_step'], d['roofline']['phase_ms_per_step'], d['roofline']['frac'])"
done
env SNN_TRACE_DEBUG=0 timeout 300 python scripts/trace.py 3 0 2>&1 | grep -v "^{" | tail -3
