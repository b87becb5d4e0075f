# compute-sanitizer over a small plastic network (graph replay + PDL, read-out
# flush): memcheck, racecheck (shared memory), synccheck; summary lines only
python -c "import __graft_entry__ as g; g.build()" || exit 1
cat > /tmp/san_run.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import workloads as W
from paper_2107_04092_b200 import Snn
for H, D in ((64, 2), (128, 2), (64, 15)):
    rc = W.brunel(5003, p=0.04, plastic=True, delay=D, seed=13)
    g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=128, history_bits=H)
    rc.apply(g)
    g.step(150)
    w = g.read_state("WEIGHTS")
    print("H", H, "D", D, "steps", g.t, "spikes", int(g.read_state("SPIKE_COUNT").sum()), "w_sum", float(np.sum(w)))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --show-backtrace no python /tmp/san_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^H " gpurun_out/sanitize_$tool.log | head -5
done
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize.log 2>&1; echo "== memcheck smoke rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/sanitize.log
