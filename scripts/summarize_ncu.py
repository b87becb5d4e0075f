"""Summarise a round's ncu evidence into profiles/<round>/ (run here, not on the box).

    python scripts/summarize_ncu.py gpurun_out/full_cur.ncu-rep gpurun_out/launches.csv profiles/r02 v1 [config] [flags]

Writes ncu_<tag>.json (per kernel: one --set full launch: duration, DRAM bytes,
instructions, issue/warps active, top stall reasons) + ncu_<tag>_summary.txt,
and launches_<tag>_summary.txt (per-kernel mean duration and share of the
step from the --metrics launch list; cold-cache, serialised launches)."""
import collections
import csv
import json
import subprocess
import sys

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import source_sha  # noqa: E402

rep, launches, outdir, tag = sys.argv[1:5]
CONFIG = int(sys.argv[5]) if len(sys.argv) > 5 else 3
FLAGS = sys.argv[6] if len(sys.argv) > 6 else ""
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
        "nsecond": 1e-3, "msecond": 1e3}
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed_op_shared_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"]
out, txt = {}, []
for d in rows[2:]:
    name = d[hdr.index("Kernel Name")].split("(")[0]
    k = {}
    for key in keys:
        if key not in hdr:
            continue
        v = d[hdr.index(key)].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        u = units[hdr.index(key)]
        if key.startswith("dram__bytes"):
            v *= UNIT.get(u, 1.0)
        if key == "gpu__time_duration.sum":
            v *= UNIT.get(u, 1.0)          # -> us
        k[key] = v
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(d[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    k["top_stalls"] = {h: v for v, h in sorted(st, reverse=True)[:6]}
    k["dram_bytes"] = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
    out[name] = k
    txt.append(f"== {name}")
    for key in keys:
        if key in k:
            txt.append(f"   {key:60s} {k[key]:.6g}")
    txt.append("   stall samples: " + ", ".join(f"{h}={v:g}" for h, v in k["top_stalls"].items()))
# the capture counts as bench.py's roofline.traffic only for these kernels
# (source hash), this BASELINE config and these flags
# (the hash written beside the report on the GPU box at capture time, else now)
shaf = os.path.splitext(rep)[0] + ".sha"
sha = open(shaf).read().strip() if os.path.exists(shaf) else source_sha()
out["_meta"] = {"source_sha": sha, "config": CONFIG, "flags": FLAGS, "report": os.path.basename(rep)}
json.dump(out, open(f"{outdir}/ncu_{tag}.json", "w"), indent=1)
open(f"{outdir}/ncu_{tag}_summary.txt", "w").write(
    "ncu --set full --clock-control none --import-source on, BASELINE config 3, one launch per kernel "
    "after warm-up (cold cache, serialised; durations in us, DRAM in bytes)\n" + "\n".join(txt) + "\n")

# launch list
rows = list(csv.reader(open(launches)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for d in data:
    v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
    agg[d["Kernel Name"].split("(")[0]][d["Metric Name"]].append(v)
tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
lines = [os.environ.get("NCU_LAUNCH_CMD",
                        "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                        "--clock-control none -k regex:\"k_front|k_deliver|k_flush\" -s 9000 -c 300 on `python bench.py --steps 200 "
                        "--warmup 20 --settle 3000 --no-cpu-baseline --no-e2e --no-ktime` (scripts/gpu_evidence.sh)")
         + " (graph replay; cold-cache, serialised)"]
for k, m in agg.items():
    t = m["gpu__time_duration.sum"]
    lines.append(f"{k:20s} launches={len(t):4d} mean_us={sum(t) / len(t):8.2f} share={sum(t) / tot:.3f} "
                 f"dram_read_MB={sum(m['dram__bytes_read.sum']) / len(t) / 1e6:7.2f} "
                 f"dram_write_MB={sum(m['dram__bytes_write.sum']) / len(t) / 1e6:7.2f}")
open(f"{outdir}/launches_{tag}_summary.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
print("\n".join(txt))
