# delivery tuning sweep: elements in flight per thread (kDelU) x CTAs per SM
for v in "8 2" "12 1" "16 1" "12 2"; do
  set -- $v
  SNN_NVCC_EXTRA="-DSNN_DEL_U=$1 -DSNN_DEL_MINB=$2" python -c "
import sys; sys.path.insert(0, 'paper_2107_04092_b200'); import build_ext; build_ext.build(force=True)" > /dev/null 2>&1 || { echo build failed $v; continue; }
  timeout 300 python bench.py --steps 3000 --warmup 300 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('U=$1 minB=$2 ms/step', d['ms_per_step'], d['roofline']['phase_ms_per_step']['DELIVERY'])"
done
