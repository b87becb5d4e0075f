# A/B of compile-time variants: bash scripts/gpu_variants.sh "" "-DSNN_X=1" ...
# (each: rebuild with SNN_NVCC_EXTRA, GPU tests, one config-3 bench line)
for v in "$@"; do
  SNN_NVCC_EXTRA="$v" python paper_2107_04092_b200/build_ext.py --force > gpurun_out/build_variant.log 2>&1 || { echo "BUILD FAIL [$v]"; tail -5 gpurun_out/build_variant.log; continue; }
  r=$(timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)
  timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', '$r', 'us/step', round(d['ms_per_step']*1e3,2), {k: round(v*1e3,2) for k,v in d['roofline']['phase_ms_per_step'].items() if k in ('FRONT','STDP','DELIVERY')})"
done
