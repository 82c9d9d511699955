"""Top stalled SASS instructions of an ncu report (source page) with context (not product)."""
import csv, subprocess, sys

rep = sys.argv[1]
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iall] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -float(data[i][iall] or 0))[:n_top]
for i in order:
    r = data[i]
    ctx = " | ".join(x[isrc].strip()[:50] for x in data[max(0, i - 3):i])
    print(f"{float(r[iall]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:60]:60s}  <- {ctx}")
