# step-graph structure experiments (SNN_PIPE etc., engine.cu): one short bench each.
# PIPES="name:ENV=1,ENV2=2 name2:..." (default: the serial / side-branch set)
python -c "import __graft_entry__ as g; g.build()" || exit 1
PIPES=${PIPES:-"serial: side1:SNN_PIPE=1,SNN_FL_LAG=1 side2:SNN_PIPE=1,SNN_FL_LAG=2 arrside:SNN_PIPE=2 legacy:SNN_NO_AHEAD=1"}
for cfg in $PIPES; do
  name=${cfg%%:*}; envs=${cfg#*:}; envs=${envs//,/ }
  env $envs timeout 300 python bench.py --steps ${VSTEPS:-3000} --warmup 300 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/pipe_$name.json 2> gpurun_out/pipe_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/pipe_{n}.json").read().strip().splitlines()[-1])
    ks = d["kernel_spans"]
    print(f"PIPE {n}: {d['ms_per_step']*1e3:.2f} us/step  " + " ".join(f"{k}={ks[k]['us_from_wait']:.2f}" for k in ks if isinstance(ks[k], dict)))
except Exception as e:
    print("PIPE", n, "failed", e, open(f"gpurun_out/pipe_{n}.err").read()[-400:])
PY
done
