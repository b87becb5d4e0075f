"""Per-source-line instructions executed and stall samples of one kernel in an
ncu report (--page source, cuda+sass correlation): the top lines."""
import csv, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname = None
rows = []
hdr = None
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] == "" or rec[0] == "Function Name":
        continue
    d = dict(zip(hdr[:2] + hdr[4:], rec[:2] + rec[4:]))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    rows.append((fname, int(rec[0]), rec[1].strip()[:90], ins, smp))
tot_i = sum(r[3] for r in rows)
tot_s = sum(r[4] for r in rows)
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[3]:9d} {100*r[3]/max(tot_i,1):5.1f}%  smp {r[4]:5d} {100*r[4]/max(tot_s,1):5.1f}%  {r[0]}:{r[1]}  {r[2]}")
