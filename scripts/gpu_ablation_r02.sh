# SURVEY 8(f2) ablation on BASELINE config 3 with the round-2 kernels: the
# paper's STDP schedules (Fig. 2a naive / 2b lazy / 2c event) and delivery
# kernels (Fig. 3a row-wise / 3b sliced), H = 64 / 128, 16-bit ids.
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for args in "--plasticity event" "--plasticity lazy" "--plasticity naive" "--delivery rowwise" "--history-bits 128" "--idx16"; do
  timeout 900 python bench.py --steps ${ABL_STEPS:-1000} --warmup 100 --no-cpu-baseline --no-e2e $args > gpurun_out/abl.json 2> gpurun_out/abl.err
  python - "$args" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abl.json").read().strip().splitlines()[-1])
    print(json.dumps({"args": sys.argv[1], "us_per_step": d["ms_per_step"] * 1e3, "wall_s_per_bio_s": d["value"],
                      "events_per_s": d["events_per_s"], "kernel_spans": d.get("kernel_spans"),
                      "per_step": d["per_step"], "clocks": d["clocks"]}))
except Exception as e:
    print(json.dumps({"args": sys.argv[1], "error": str(e), "stderr": open("gpurun_out/abl.err").read()[-400:]}))
PY
done > gpurun_out/ablation_r02.jsonl
python -c "
import json
for l in open('gpurun_out/ablation_r02.jsonl'):
    d = json.loads(l); print(d['args'], round(d.get('us_per_step', -1), 2), d.get('error', ''))"
