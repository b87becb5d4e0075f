"""Per-CTA %globaltimer marks of the graph-replayed step (SNN_FLAG_TRACE with
SNN_TRACE_GRAPH: the last step of a 64-step graph), saved for offline reading."""
import sys, os
os.environ["SNN_TRACE_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads as W
from paper_2107_04092_b200 import Snn, FLAG_TRACE

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace_graph.npy"
rc = W.config(cfg)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=0, flags=FLAG_TRACE)
rc.apply(g)
g.step(3008)
torch.cuda.synchronize()
reps = []
for rep in range(4):
    g.step(64)
    torch.cuda.synchronize()
    reps.append(g.read_state("TRACE").reshape(4, 4096, 4).astype(np.int64))
np.save(out, np.stack(reps))
for tr in reps:
    t0 = tr[0][tr[0][:, 0] > 0][:, 0].min()
    for k, name in [(0, "front"), (2, "deliver"), (3, "flush")]:
        a = tr[k][tr[k][:, 0] > 0]
        rel = (a - t0) / 1000.0
        print(f"{name:8s} ctas={len(a):4d} start[min/med/max]={rel[:,0].min():7.2f}/{np.median(rel[:,0]):7.2f}/{rel[:,0].max():7.2f} "
              + " ".join(f"ph{p}[med/max]={np.median(rel[:,p]-rel[:,0]):6.2f}/{(rel[:,p]-rel[:,0]).max():6.2f}" for p in (1, 2, 3))
              + f" end[med/max]={np.median(rel[:,3]):7.2f}/{rel[:,3].max():7.2f}")
