"""First step at which the GPU raster departs from the oracle's, and the long-run
rate / weight-histogram differences (Brunel+ 31,623, seed 3, 10,000 steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from oracle.oracle import Oracle
from paper_2107_04092_b200 import Snn
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rc = W.brunel(31_623, p=0.02, plastic=True, delay=15, seed=seed)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
rc.apply(g)
o = Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
rc.apply(o)
o.finalize(); g.finalize()
first = None
done = 0
while done < steps:
    n = 50 if first is None else steps - done
    g.step(n); o.step(n); done += n
    if first is None and not np.array_equal(g.read_state("HIST"), o.array("hist")):
        first = done
sg = g.read_state("SPIKE_COUNT").astype(np.float64); so = o.array("nspk").astype(np.float64)
b = 0; out = []
for p in rc.pops:
    out.append(f"{p.name} {100 * (sg[b:b+p.n].sum() - so[b:b+p.n].sum()) / so[b:b+p.n].sum():+.2f}%")
    b += p.n
print(f"mode {os.environ.get('SNN_NO_AHEAD', 'ahead')} seed {seed}: rasters equal up to step ~{first}; rates", " ".join(out))
