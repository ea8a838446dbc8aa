"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): mean duration per
kernel, full-size launches and the z-slab launches of the host-buffer applies separately,
and the momentum / pressure share of a bench step.  usage: ncu_launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
by = collections.defaultdict(list)
for r in rows[1:]:
    by[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
full, slab = {}, {}
for k, v in by.items():
    big = [t for t in v if t > 0.5 * max(v)]
    small = [t for t in v if t <= 0.5 * max(v)]
    full[k] = big
    if small:
        slab[k] = small
print("## full-size launches")
for k, v in full.items():
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v) / len(v):9.1f} us")
print("## e2e z-slab launches")
for k, v in slab.items():
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v) / len(v):9.1f} us")
mom = [sum(v) / len(v) for k, v in full.items() if "k_momentum" in k]
prs = [sum(v) / len(v) for k, v in full.items() if "k_sip" in k]
if mom and prs:
    t = mom[0] + prs[0]
    print(f"## share of a bench step (one momentum + one pressure apply): momentum {100 * mom[0] / t:.1f} %, "
          f"pressure {100 * prs[0] / t:.1f} %")
