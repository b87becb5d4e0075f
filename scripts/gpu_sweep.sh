# build + bench of variants: RUNS="name|nvcc flags (comma-separated)|env assignments (comma-separated)" ...
# then (TESTS=1) the GPU tests on the default build
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
if [ -n "$TESTS" ]; then
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
  timeout 900 python -m pytest tests -m gpu -x -q ${PYT_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
  tail -5 gpurun_out/pytest_gpu.log
fi
last="__none__"
for r in $RUNS; do
  name=$(echo "$r" | cut -d'|' -f1); flags=$(echo "$r" | cut -d'|' -f2); envs=$(echo "$r" | cut -d'|' -f3)
  flags=${flags//,/ }; envs=${envs//,/ }
  if [ "$flags" != "$last" ]; then
    rm -f paper_2107_04092_b200/libsnn.so
    SNN_NVCC_EXTRA="$flags" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
    last="$flags"
  fi
  env $envs timeout 300 python bench.py --steps ${VSTEPS:-3000} --warmup 300 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{n}.json").read().strip().splitlines()[-1])
    ks = d["kernel_spans"]
    print(f"VARIANT {n}: us/step {d['ms_per_step']*1e3:.2f}  " + " ".join(f"{k}={ks[k]['us_from_wait']:.2f}/{ks[k]['us_from_entry']:.2f}" for k in ks if isinstance(ks[k], dict)) + f" frac={d['roofline']['frac']:.3f} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print("VARIANT", n, "failed", e, open(f"gpurun_out/var_{n}.err").read()[-800:])
PY
done
rm -f paper_2107_04092_b200/libsnn.so
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
