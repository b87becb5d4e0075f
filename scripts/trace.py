"""Per-CTA phase trace of simulation steps (debug, SNN_FLAG_TRACE; direct launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json as _json
import numpy as np
import torch
import workloads as W
from paper_2107_04092_b200 import Snn, FLAG_TRACE

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
C = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rc = W.config(cfg)
extra = int(os.environ.get("SNN_TRACE_FLAGS", "0"))
kw = _json.loads(os.environ.get("SNN_TRACE_KW", "{}"))      # e.g. {"flush_period": 16}
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=C, flags=FLAG_TRACE | extra, **kw)
rc.apply(g)
g.step(int(os.environ.get("SNN_TRACE_T0", "3000")))
torch.cuda.synchronize()
dbg = os.environ.get("SNN_TRACE_DEBUG")
for rep in range(3):
    if dbg is not None:
        os.environ["SNN_DEBUG_KERNELS"] = dbg     # kernel experiment on the traced steps only
    g.step(1)
    os.environ.pop("SNN_DEBUG_KERNELS", None)
    tr = g.read_state("TRACE").reshape(4, 4096, 4).astype(np.int64)
    t0 = tr[0][tr[0][:, 0] > 0][:, 0].min()
    for k, name in [(0, "front"), (2, "deliver"), (1, "stdp"), (3, "flush")]:
        a = tr[k]
        a = a[a[:, 0] > 0]
        if len(a) == 0:
            continue
        rel = (a - t0) / 1000.0
        print(f"{name:8s} ctas={len(a):4d} start[min/med/max]={rel[:,0].min():7.2f}/{np.median(rel[:,0]):7.2f}/{rel[:,0].max():7.2f} "
              + " ".join(f"ph{p}[med/max]={np.median(rel[:,p]-rel[:,0]):6.2f}/{(rel[:,p]-rel[:,0]).max():6.2f}" for p in (1, 2, 3))
              + f" end_max={rel[:,3].max():7.2f}")
    print(g.metrics())
# deliver: element-phase duration by slice (E slices carry the plastic arrivals' STDP in the ahead step)
a = tr[2][:g.info()["nslices"] * 2] if False else None
tr = g.read_state("TRACE").reshape(4, 4096, 4).astype(np.int64)
ns = g.info()["nslices"]
d = tr[2][: ns * 2]
ok = d[:, 0] > 0
ph = (d[:, 2] - d[:, 1]) / 1000.0
cta = np.arange(len(d))
sl = cta % ns                      # blockIdx.y * gridDim.x + blockIdx.x
nE = rc.pops[0].n
C = g.info()["C"]
isE = (sl + 1) * C <= nE
print("deliver element phase (us): E slices med/max %.2f/%.2f   other slices med/max %.2f/%.2f" %
      (np.median(ph[ok & isE]), ph[ok & isE].max(), np.median(ph[ok & ~isE]), ph[ok & ~isE].max()))
