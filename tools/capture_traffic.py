"""Roofline traffic on HEAD (committed recipe): parse an ncu launch list with
gpu__time_duration / dram__bytes_read / dram__bytes_write (tools/gpu/traffic.sh) and write the
dominant phase's per-launch DRAM bytes (layer 0 of the bench's profile-only C3 step) to
profiles/dram_bytes_per_launch.json, which bench.py reports as roofline.traffic."""
import collections, csv, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r"([A-Za-z_0-9]+)(<[^>]*>)?\(", r[ki])
    name = m.group(1) if m else r[ki][:40]
    d = launch.setdefault(int(r[ii]), {"name": name})
    d[r[mi]] = float(r[vi].replace(",", ""))
bwd_names = ("bwd_prep_kernel", "transpose_sel_kernel", "scan_kernel", "attn_bwd_dkv_kernel", "attn_bwd_dq_kernel",
             "q_records_kernel", "match_rounds_kernel", "dkv_split_kernel", "dkv_split_reduce_kernel")
first_bwd = {}
for lid, d in launch.items():  # layer 0: the first launch of every backward kernel
    if d["name"] in bwd_names and d["name"] not in first_bwd:
        first_bwd[d["name"]] = d
fwd = next(d for d in launch.values() if d["name"] == "attn_fwd2_kernel")
tot = lambda d: d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)  # noqa: E731
sha = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
out = {"c3": {"dominant_traffic_bytes": sum(tot(d) for d in first_bwd.values()),
              "per_kernel_bytes": {n: tot(d) for n, d in first_bwd.items()},
              "fwd_traffic_bytes": tot(fwd),
              "note": f"ncu launch list of `bench.py --profile-only` (C3, rank 0, layer 0's backward), "
                      f"dram__bytes_read.sum + dram__bytes_write.sum, build {sha}; tools/gpu/traffic.sh"}}
path = os.path.join(ROOT, "profiles", "dram_bytes_per_launch.json")
old = json.load(open(path)) if os.path.exists(path) else {}
old.update(out)
json.dump(old, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
