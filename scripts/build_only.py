"""Build the BASELINE config-3 graph a few times and print the device-timed
construction (SNN_PHASE_BUILD) of each (setup path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2107_04092_b200 import Snn
rc = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
    rc.apply(g)
    g.step(1)
    torch.cuda.synchronize()
    ms = g.phase_times()["BUILD"]
    S = g.info()["S"]
    print(f"build {ms:.2f} ms, {S} synapses, {S / ms:.3e} synapses/ms")
    del g
    torch.cuda.empty_cache()
