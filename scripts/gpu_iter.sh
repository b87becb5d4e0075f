# iteration check: build, GPU parity tests, per-CTA phase trace, short bench
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/trace.py 3 0 > gpurun_out/trace.log 2>&1; echo trace=$?
tail -4 gpurun_out/trace.log
timeout 300 python bench.py --steps 3000 --warmup 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("ms/step", d["ms_per_step"], "value", d["value"], "frac", r["frac"], "phase", r["phase_ms_per_step"], "kern", {k: v["achieved_gbs"] for k, v in r["kernels"].items()})
PY
if [ -n "$ALT_ENV" ]; then
env $ALT_ENV timeout 300 python bench.py --steps 3000 --warmup 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_alt.json 2> gpurun_out/bench_alt.err; echo bench_alt=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_alt.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("ALT ms/step", d["ms_per_step"], "frac", r["frac"], "phase", r["phase_ms_per_step"])
PY
fi
