# iteration check: build, GPU parity tests, the driver's bench command, a longer bench
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout ${PYT_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYT_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; echo bench_driver=$?
tail -3 gpurun_out/bench_driver.err
timeout 600 python bench.py --steps ${ITER_STEPS:-3000} --warmup 300 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench=$?
tail -3 gpurun_out/bench_iter.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_driver.json", "gpurun_out/bench_iter.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}
    print(f, "ms/step", d["ms_per_step"], "value", d["value"], "rates", d["rates_hz"], "frac", r.get("frac"),
          "kern", {k: (round(v["us_per_launch"], 2), round(v["achieved_gbs"])) for k, v in (r.get("kernels") or {}).items()},
          "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"),
          "spans", d.get("kernel_spans"))
PY
