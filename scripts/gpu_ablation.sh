# SURVEY 8(f2) ablation on BASELINE config 3: plasticity schedules x delivery kernels, H = 64 / 128
python -c "import __graft_entry__ as g; g.build()" || exit 1
for args in "--plasticity event" "--plasticity lazy" "--plasticity naive" "--delivery rowwise" "--history-bits 128"; do
  timeout 600 python bench.py --steps ${ABL_STEPS:-1000} --warmup 200 --phase-steps 200 --no-cpu-baseline --no-e2e $args > gpurun_out/abl.json 2> gpurun_out/abl.err
  python - "$args" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abl.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(json.dumps({"args": sys.argv[1], "ms_per_step": d["ms_per_step"], "wall_s_per_bio_s": d["wall_s_per_bio_s"],
                  "events_per_s": d["value"], "phase_ms_per_step": r["phase_ms_per_step"],
                  "per_step": d["per_step"], "clocks": d["clocks"]}))
PY
done > gpurun_out/ablation.jsonl
cat gpurun_out/ablation.jsonl
