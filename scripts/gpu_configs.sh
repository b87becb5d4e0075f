# every BASELINE config on one GPU (short runs): completes, and the numbers
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 2000 --warmup 200 --phase-steps 200 --no-cpu-baseline --no-e2e > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/cfg{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("cfg", c, "FAILED", open(f"gpurun_out/cfg{c}.err").read()[-500:]); sys.exit(0)
r = d["roofline"]
print(json.dumps({"config": c, "workload": d["config"]["workload"], "synapses": d["config"]["synapses"],
                  "slice_width": d["config"]["slice_width"], "ms_per_step": d["ms_per_step"],
                  "wall_s_per_bio_s": d["wall_s_per_bio_s"], "events_per_s": d["value"],
                  "phase_ms_per_step": {k: v for k, v in r["phase_ms_per_step"].items() if k in ("FRONT", "STDP", "DELIVERY")},
                  "dominant": r["kernel"], "frac": r["frac"], "setup_build_ms": d["setup"]["build_ms"],
                  "rates_hz": d["rates_hz"]}))
PY
done > gpurun_out/configs.jsonl
cat gpurun_out/configs.jsonl
