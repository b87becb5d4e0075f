import sys, os, faulthandler
faulthandler.enable()
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads as W
from oracle import oracle as O
from paper_2107_04092_b200 import Snn
rc = W.brunel(10000, p=0.05, plastic=True, delay=0, seed=7)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=512)
rc.apply(g)
g.finalize()
o = O.Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, threads=8)
rc.apply(o)
o.finalize()
print("rowptr eq", np.array_equal(g.read_state("ROW_PTR"), o.array("row_ptr")), flush=True)
print("idx eq", np.array_equal(g.read_state("IDX"), o.array("idx")), flush=True)
w0 = g.read_state("WEIGHTS")
print("w0 eq", np.array_equal(w0, o.array("w")), w0[:5], o.array("w")[:5], flush=True)
for t in range(70):
    g.step(1); o.step(1)
    if t in (0, 1, 10, 62, 63, 64, 69):
        w = g.read_state("WEIGHTS")
        bad = np.abs(w - o.array("w")) > 1e-4 * np.maximum(np.abs(o.array("w")), 1e-2)
        print(t, "bad", int(bad.sum()), np.flatnonzero(bad)[:5], w[bad][:5], o.array("w")[bad][:5], flush=True)
print("metrics", g.metrics(), flush=True)
print("STEP", g.read_state("STEP"), flush=True)
print("INFO try", flush=True)
print(g.info(), flush=True)
