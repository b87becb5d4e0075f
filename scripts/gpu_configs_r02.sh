# every BASELINE config on one GPU with the round-2 kernels (short runs after the settle)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 2000 --warmup 200 --no-cpu-baseline --no-e2e > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/cfg{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(json.dumps({"config": c, "error": open(f"gpurun_out/cfg{c}.err").read()[-500:]})); sys.exit(0)
r = d.get("roofline") or {}
print(json.dumps({"config": c, "workload": d["config"]["workload"], "synapses": d["config"]["synapses"],
                  "slice_width": d["config"]["slice_width"], "us_per_step": d["ms_per_step"] * 1e3,
                  "wall_s_per_bio_s": d["value"], "events_per_s": d["events_per_s"],
                  "kernel_spans": d.get("kernel_spans"), "dominant": r.get("kernel"), "frac": r.get("frac"),
                  "build_ms": d["setup"]["build_ms"], "rates_hz": d["rates_hz"]}))
PY
done > gpurun_out/configs_r02.jsonl
python -c "
import json
for l in open('gpurun_out/configs_r02.jsonl'):
    d = json.loads(l); print(d['config'], d.get('workload'), round(d.get('us_per_step', -1), 2), d.get('dominant'), d.get('build_ms'), d.get('error', '')[:200])"
