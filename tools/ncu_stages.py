"""Stall / smem / instruction share per kernel stage (stage markers are '// X:' comments)."""
import csv, collections, subprocess, re, sys
rep, kern, src_path = sys.argv[1], sys.argv[2], sys.argv[3]
first = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iW = hdr.index("L1 Wavefronts Shared"); iI = hdr.index("Instructions Executed")
src = open(src_path).read().split("\n")
marks = [(i + 1, m.group(1)) for i, l in enumerate(src) if i >= first and (m := re.match(r"\s*// (S\d|[A-D]|F\d|-+ \w+)", l))]
def stage(ln):
    s = "pre"
    for l, n in marks:
        if ln >= l: s = n
    return s if ln >= first else "helpers"
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
def f(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0].strip().isdigit(): continue
    a = agg[stage(int(r[0]))]
    a[0] += f(r[iS]); a[1] += f(r[iW]); a[2] += f(r[iI])
ts, tw, ti = (sum(v[k] for v in agg.values()) or 1 for k in range(3))
for k, v in agg.items():
    print(f"{k[:20]:20s} stall {100*v[0]/ts:5.1f}%  smem {100*v[1]/tw:5.1f}%  inst {100*v[2]/ti:5.1f}%")
