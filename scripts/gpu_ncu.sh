# one ncu --set full capture of the step kernels (BASELINE config, after the
# settle steps), individual launches; the source hash is written beside it
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import bench; print(bench.source_sha())" > gpurun_out/full_cur.sha
cat > /tmp/prof_run.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2107_04092_b200 import Snn
rc = W.config(int(os.environ.get("NCU_CONFIG", "3")))
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, flags=int(os.environ.get("NCU_FLAGS", "1")))   # 1 = NO_GRAPH: individual launches; 0 = graph nodes
rc.apply(g)
g.step(int(os.environ.get("NCU_STEPS", "3200")))
torch.cuda.synchronize()
PY
KREGEX=${KREGEX:-"k_deliver|k_stdp|k_front"}
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${NSKIP:-9300} -c ${NCOUNT:-3} -o gpurun_out/full_cur -f python /tmp/prof_run.py > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
