# one ncu --set full capture of k_deliver and k_stdp (config 3, after warm-up)
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
ncu --set full --clock-control none --import-source on -k regex:"k_deliver|k_stdp" -s 2900 -c 2 -o gpurun_out/full_cur python /tmp/prof_run.py > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
