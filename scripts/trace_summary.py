"""Summary of a per-CTA trace of graph-replayed steps (scripts/trace_graph.py
output, [reps][kernel][cta][mark] %globaltimer ns): per kernel the CTA start /
end percentiles and per-CTA phase durations, t = 0 at the first k_front CTA.
Marks: k_front 0 entry, 3 end; k_deliver 0 entry, 1 return from the
dependency wait, 2 elements done, 3 end; k_flush 0 entry, 1/2 table copy
wait, 3 end.  (k_deliver CTA = split * nslices + slice.)"""
import sys
import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace_graph.npy"
r = np.load(path)
pct = [0, 10, 50, 90, 100]
for rep, tr in enumerate(r):
    t0 = tr[0][tr[0][:, 0] > 0][:, 0].min()
    print(f"-- step {rep} (the last step of a 64-step graph; us)")
    for k, name in [(0, "k_front"), (2, "k_deliver"), (3, "k_flush")]:
        a = tr[k][tr[k][:, 0] > 0]
        if len(a) == 0:
            continue
        rel = (a - t0) / 1000.0
        print(f"  {name:9s} ctas {len(a):4d}  start p{pct} {np.percentile(rel[:, 0], pct).round(1).tolist()}"
              f"  end {np.percentile(rel[:, 3], pct).round(1).tolist()}  duration med {np.median(rel[:, 3] - rel[:, 0]):.1f}")
        if k == 2:
            print(f"  {'':9s} wait returns {np.percentile(rel[:, 1], pct).round(1).tolist()}"
                  f"  elements after the wait med {np.median(rel[:, 2] - rel[:, 1]):.1f}")
