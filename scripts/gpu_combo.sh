# (compile flags x env) combinations, one short bench each: COMBOS="name|-DX=1,-DY=2|ENV=1 ENV2=3 ..."
for c in $COMBOS; do
  name=${c%%|*}; rest=${c#*|}; flags=${rest%%|*}; envs=${rest#*|}; flags=${flags//,/ }; envs=${envs//,/ }
  rm -f paper_2107_04092_b200/libsnn.so
  SNN_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  env $envs timeout 300 python bench.py --steps ${VSTEPS:-3000} --warmup 300 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/combo_$name.json 2> gpurun_out/combo_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/combo_{n}.json").read().strip().splitlines()[-1])
    ks = d["kernel_spans"]
    print(f"COMBO {n}: {d['ms_per_step']*1e3:.2f} us/step  " + " ".join(f"{k}={ks[k]['us_from_wait']:.2f}" for k in ks if isinstance(ks[k], dict)))
except Exception as e:
    print("COMBO", n, "failed", e, open(f"gpurun_out/combo_{n}.err").read()[-400:])
PY
done
rm -f paper_2107_04092_b200/libsnn.so
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
