"""Shared-memory bank-conflict simulator for qp_sip_field (fast_deformed.cuh): the cell
stages C1-C5 and face stages F1-F5 of the deformed SIP operator (k_sip_qp, and pass A of
k_momentum_qp), one warp per cell.  Model as tools/bank_sim_sip1.py (64-bit accesses:
two half-warps; wavefronts = max distinct addresses per 8-byte bank slot, a % 16), which
reproduced ncu's per-line excess wavefronts.

Layout parameters searched (strides in doubles, defaults = the round-1 layout):
  SQX  stride of qx in the [qx][k][j] x-pass arrays (XB, XD, P2, R02)      default N*N
  SR   stride of r = qx*Q + qy in the [r][k] arrays (YBB.., PP..)         default N
  SKR  stride of k in those arrays                                        default 1
  SFL  per-field stride of the F1/F2 trace arrays (fl)                    default N*N
  SFQ  q stride inside fl                                                 default N
  SFP  F2 -> F3 array: stride of q (fp[fld][q][qp])                       default Q
  SFA  F3 -> F4 array: stride of qp (fa[part][qp][b])                     default N
  SFO  F4 -> F5 array: stride of bq (fo[bp + SFO * bq])                   default N
usage: python tools/bank_sim_qp.py N Q"""
import itertools
import sys


def wav(addrs):
    tot = 0
    for h in (0, 1):
        banks = {}
        for ln, a in addrs:
            if ln // 16 != h:
                continue
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


def sim(N, Q, SQX=None, SR=None, SKR=1, SFL=None, SFQ=None, SFP=None, SFA=None, SFO=None, report=False):
    NF, QQ = N * N, Q * Q
    SQX = SQX or NF
    SR = SR or N
    SFL = SFL or NF
    SFQ = SFQ or N
    SFP = SFP or Q
    SFA = SFA or N
    SFO = SFO or N
    XB = 0
    XD = XB + Q * SQX + 1
    YB = 0  # separate regions: conflicts only depend on strides within one array
    FL, FP, FA, FO = 0, 0, 0, 0
    per_stage = {}

    def run(name, nitems, fn):
        tot = 0
        for rnd in range((nitems + 31) // 32):
            insts = {}
            for lane in range(32):
                it = lane + 32 * rnd
                if it >= nitems:
                    continue
                for key, a in fn(it):
                    insts.setdefault(key, []).append((lane, a))
            for ad in insts.values():
                tot += wav(ad)
        per_stage[name] = tot

    cell = lambda i, j, k: i + N * j + NF * k
    xq = lambda qx, j, k: qx * SQX + j + N * k
    rk = lambda r, k: r * SR + k * SKR
    run("C1", NF, lambda jk: [(("r", i), cell(i, jk % N, jk // N)) for i in range(N)] +
        [(("w", qx), xq(qx, jk % N, jk // N)) for qx in range(Q)])
    run("C2", Q * N, lambda it: [(("r", j), xq(it // N, j, it % N)) for j in range(N)] +
        [(("w", qy), rk((it // N) * Q + qy, it % N)) for qy in range(Q)])
    run("C3", QQ, lambda r: [(("r", k), rk(r, k)) for k in range(N)] + [(("w", k), rk(r, k)) for k in range(N)])
    run("C4", Q * N, lambda it: [(("r", qy), rk((it // N) * Q + qy, it % N)) for qy in range(Q)] +
        [(("w", j), xq(it // N, j, it % N)) for j in range(N)])
    run("C5", NF, lambda jk: [(("r", qx), xq(qx, jk % N, jk // N)) for qx in range(Q)] +
        [(("w", i), cell(i, jk % N, jk // N)) for i in range(N)])

    def strides(a):
        sl = 1 if a == 0 else (N if a == 1 else NF)
        sp = N if a == 0 else 1
        sq = N if a == 2 else NF
        return sl, sp, sq

    def F1(it):
        f, tn = divmod(it, NF)
        a = f >> 1
        p, q = tn % N, tn // N
        sl, sp, sq = strides(a)
        base = p * sp + q * sq
        out = [(("U", l), base + l * sl) for l in range(N)]
        out += [(("fl", fld), f * 4 * SFL + fld * SFL + p + SFQ * q) for fld in range(4)]
        return out
    run("F1", 6 * NF, F1)

    def F2(it):
        f, q = divmod(it, N)
        out = [(("fl", fld, p), f * 4 * SFL + fld * SFL + p + SFQ * q) for fld in range(4) for p in range(N)]
        out += [(("fp", fld, qp), f * 6 * N * SFP + fld * N * SFP + q * SFP + qp) for fld in range(6) for qp in range(Q)]
        return out
    run("F2", 6 * N, F2)

    def F3(it):
        f, qp = divmod(it, Q)
        out = [(("fp", fld, q), f * 6 * N * SFP + fld * N * SFP + q * SFP + qp) for fld in range(6) for q in range(N)]
        out += [(("fa", part, b), f * 3 * Q * SFA + part * Q * SFA + qp * SFA + b) for part in range(3) for b in range(N)]
        return out
    run("F3", 6 * Q, F3)

    def F4(it):
        f, bq = divmod(it, N)
        out = [(("fa", part, qp), f * 3 * Q * SFA + part * Q * SFA + qp * SFA + bq) for part in range(3) for qp in range(Q)]
        out += [(("fo", h, bp), f * 2 * N * SFO + h * N * SFO + bp + SFO * bq) for h in range(2) for bp in range(N)]
        return out
    run("F4", 6 * N, F4)

    def F5(a):
        def fn(tn):
            p, q = tn % N, tn // N
            out = [(("f0", 0), (2 * a) * 2 * N * SFO + N * SFO + p + SFO * q), (("f1", 0), (2 * a + 1) * 2 * N * SFO + N * SFO + p + SFO * q)]
            sl, sp, sq = strides(a)
            out += [(("o", l), l * sl + p * sp + q * sq) for l in range(N)]
            return out
        return fn
    for a in range(3):
        run(f"F5{a}", NF, F5(a))
    tot = sum(per_stage.values())
    if report:
        print(per_stage)
    return tot


if __name__ == "__main__":
    N, Q = int(sys.argv[1]), int(sys.argv[2])
    NF = N * N
    base = sim(N, Q, report=True)
    print("round-1 layout:", base)
    best = {}
    for name, rng in (("SQX", range(NF, NF + 17)), ("SR", range(N, N + 9)), ("SFL", range(NF, NF + 17)),
                      ("SFQ", range(N, N + 5)), ("SFP", range(Q, Q + 9)), ("SFA", range(N, N + 9)), ("SFO", range(N, N + 9))):
        res = sorted((sim(N, Q, **{**best, name: v}), v) for v in rng)
        best[name] = res[0][1]
    # second pass (interactions)
    for name, rng in (("SQX", range(NF, NF + 17)), ("SR", range(N, N + 9)), ("SFL", range(NF, NF + 17)),
                      ("SFQ", range(N, N + 5)), ("SFP", range(Q, Q + 9)), ("SFA", range(N, N + 9)), ("SFO", range(N, N + 9))):
        res = sorted((sim(N, Q, **{**best, name: v}), v) for v in rng)
        best[name] = res[0][1]
    print("best:", best, sim(N, Q, **best, report=True))
