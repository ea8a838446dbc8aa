"""Per-stage instruction mix / stall reasons of k_momentum_axis from an ncu report
(--page source --print-source cuda,sass): SASS rows are attributed to the source line
above them, lines to the kernel stage whose marker comment precedes them.
usage: python tools/ncu_stage_mix.py report.ncu-rep [kernel-regex] [fast_axis.cuh of the captured build]"""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_momentum_axis"
src = sys.argv[3] if len(sys.argv) > 3 else "paper_2107_07776_b200/csrc/fast_axis.cuh"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
col = {n: h.index(n) for n in ("Instructions Executed", "Thread Instructions Executed",
                               "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared")}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
lines = open(src).read().split("\n")
# stage markers: (first line, name)
marks = []
kstart = next(i for i, t in enumerate(lines, 1) if "k_momentum_axis(MeshArgs" in t)
for i, t in enumerate(lines, 1):
    m = re.search(r"//\s*(?:-+\s*)?(S0|A|B|C|D|F1|F2|F3|S45|S6|S78|store|pass A|pass B cell|LF advective)\b", t)
    if m and i >= kstart:
        marks.append((i, m.group(1)))
def stage(ln):
    if ln < 0: return "other-files"
    if ln < kstart: return "helpers"
    name = "pre"
    for i, n in marks:
        if i <= ln: name = n
    return name
f = lambda x: float(x.replace(",", "") or 0) if x not in ("-", "") else 0.0
agg = collections.defaultdict(lambda: collections.Counter())
cur = None
infile = True
for r in rows[hi + 1:]:
    if r and r[0] == "File Path":
        infile = r[1].endswith("fast_axis.cuh"); continue
    if len(r) < len(h) or r[0] == "Line No": continue
    if r[0].strip().isdigit():
        cur = int(r[0]) if infile else -1; continue
    if cur is None or not r[3].strip(): continue
    op = r[3].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    a = agg[stage(cur)]
    wi = f(r[col["Instructions Executed"]])
    a["inst"] += wi
    a["lanes"] += f(r[col["Thread Instructions Executed"]])
    a["fp64"] += wi if o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX") else 0
    a["lds_sts"] += wi if o in ("LDS", "STS") else 0
    a["ldc"] += wi if o.startswith("LDC") else 0
    a["int_ctl"] += wi if o in ("IMAD", "ISETP", "BRA", "BSSY", "BSYNC", "LOP3", "VIADD", "SHF", "LEA", "SEL", "IADD3", "PLOP3", "PRMT", "IMNMX") else 0
    a["stall"] += f(r[col["Warp Stall Sampling (All Samples)"]])
    for s in stalls:
        a[s] += f(r[h.index(s)])
tot_i = sum(a["inst"] for a in agg.values()); tot_s = sum(a["stall"] for a in agg.values())
print(f"{'stage':12s} {'inst%':>6s} {'stall%':>6s} {'lanes':>5s} {'fp64%':>6s} {'lds/sts%':>8s} {'ldc%':>5s} {'int/ctl%':>8s}  top stalls")
order = ["helpers", "pre", "S0", "pass A", "A", "B", "C", "D", "LF advective", "F1", "F2", "F3", "pass B cell", "S45", "S6", "S78", "store"]
for st in sorted(agg, key=lambda s: order.index(s) if s in order else 99):
    a = agg[st]
    top = sorted(((a[s], s[6:]) for s in stalls), reverse=True)[:3]
    ts = ", ".join(f"{n} {100 * v / max(a['stall'], 1):.0f}%" for v, n in top)
    print(f"{st:12s} {100*a['inst']/tot_i:6.1f} {100*a['stall']/tot_s:6.1f} {a['lanes']/max(a['inst'],1):5.1f} "
          f"{100*a['fp64']/max(a['inst'],1):6.1f} {100*a['lds_sts']/max(a['inst'],1):8.1f} {100*a['ldc']/max(a['inst'],1):5.1f} "
          f"{100*a['int_ctl']/max(a['inst'],1):8.1f}  {ts}")
