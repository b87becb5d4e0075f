# one ncu --set full capture of the step kernels (config 3, after warm-up), individual launches
python -c "import __graft_entry__ as g; g.build()" || exit 1
cat > /tmp/prof_run.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2107_04092_b200 import Snn
rc = W.config(3)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, flags=1)   # NO_GRAPH: individual launches
rc.apply(g)
g.step(1500)
torch.cuda.synchronize()
PY
KREGEX=${KREGEX:-"k_deliver|k_stdp|k_front"}
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${NSKIP:-4400} -c ${NCOUNT:-3} -o gpurun_out/full_cur -f python /tmp/prof_run.py > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
