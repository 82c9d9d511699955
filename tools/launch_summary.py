"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel count, total, share."""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r"([A-Za-z_0-9]+)(<[^>]*>)?\(", r[ki])
    name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:50]
    try:
        agg[name].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'n':>5s} {'total us':>11s} {'share':>6s} {'mean us':>9s}")
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{n[:48]:48s} {len(v):5d} {sum(v) / 1e3:11.1f} {sum(v) / tot:6.3f} {sum(v) / len(v) / 1e3:9.1f}")
