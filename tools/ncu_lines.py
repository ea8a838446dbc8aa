"""Per-source-line stall samples / smem wavefronts for one kernel of an ncu report."""
import csv, collections, subprocess, sys
rep, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
iW = hdr.index("L1 Wavefronts Shared"); iWE = hdr.index("L1 Wavefronts Shared Excessive")
agg = collections.defaultdict(lambda: [0.0] * 4)
def f(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0].strip().isdigit(): continue
    a = agg[int(r[0])]
    a[0] += f(r[iS]); a[1] += f(r[iI]); a[2] += f(r[iW]); a[3] += f(r[iWE])
tot = sum(v[0] for v in agg.values()) or 1
totw = sum(v[2] for v in agg.values()) or 1
lines = open(src).read().split("\n")
print(f"total stall samples {tot:.0f}, smem wavefronts {totw:.3g}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:4d} stall={100*v[0]/tot:5.1f}% inst={v[1]:.3g} wf={100*v[2]/totw:5.1f}% excess={v[3]:.3g} | {lines[ln-1].strip()[:70]}")
