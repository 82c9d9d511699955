"""Balance decomposition of a driver run (not product): per iteration, the imbalance the DST plan
itself predicts (max / mean of the per-micro-batch sums of t_final_ms in decisions_<it>.csv, the
reference's own cost of its own decisions) next to the measured busy-time imbalance
(iterations.csv). Usage: python tools/balance_decompose.py <run dir with iterations.csv>"""
import collections
import csv
import os
import sys

d = sys.argv[1]
meas = [float(r["imbalance"]) for r in csv.DictReader(open(os.path.join(d, "iterations.csv")))]
print("iter  predicted  measured")
for it, m in enumerate(meas):
    pred = collections.defaultdict(float)
    for r in csv.DictReader(open(os.path.join(d, f"decisions_{it}.csv"))):
        pred[int(r["mb"])] += float(r["t_final_ms"])
    v = list(pred.values())
    print(f"{it:4d}  {max(v) / (sum(v) / len(v)):9.3f}  {m:8.3f}")
