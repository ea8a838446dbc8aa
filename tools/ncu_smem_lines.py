"""Top source lines of a kernel by excessive (bank-conflict) shared-memory wavefronts."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
iE = hdr.index("L1 Wavefronts Shared Excessive"); iW = hdr.index("L1 Wavefronts Shared"); iS = hdr.index("Warp Stall Sampling (All Samples)")
def f(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
lines = [(f(r[iE]), f(r[iW]), f(r[iS]), r[0], r[1].strip()[:90]) for r in rows[hi + 1:] if len(r) >= len(hdr) and r[0].strip().isdigit()]
tE = sum(l[0] for l in lines) or 1; tW = sum(l[1] for l in lines) or 1
print(f"excessive {tE:.3g} of {tW:.3g} shared wavefronts")
for e, w, s, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{ln:>5s} exc {100*e/tE:5.1f}%  wav {100*w/tW:5.1f}%  stall {s:8.0f}  {src}")
