import sys, os
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2107_04092_b200 import Snn
rc = W.config(3)
g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
rc.apply(g)
g.step(1)
torch.cuda.synchronize()
print("built")
