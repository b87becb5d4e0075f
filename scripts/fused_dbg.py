"""(debug) the fused step graph under compute-sanitizer: Brunel+ 10,000, C = 512, snn_step(37) x 3."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import workloads as W
from paper_2107_04092_b200 import Snn
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rc = W.brunel(n, p=0.05, plastic=True, delay=15, seed=17)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=512)
rc.apply(g); g.finalize()
for k in range(3):
    g.step(37)
    print(k, int(g.read_state("SPIKE_COUNT").sum()), flush=True)
