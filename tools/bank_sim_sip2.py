"""Shared-memory bank-conflict simulator for k_sip_axis<2> (Q2 pressure, cfg3): the line
stages A-D of the CTA-wide (16 cells, 128 threads) variant, as tools/bank_sim_sip1.py does
for K_p = 1.  Parameters: x-pitch PX, component/array pad CTpad, cell-stride pad PERpad and
the item order (cell-major = round-1, cell-fastest).  usage: python tools/bank_sim_sip2.py"""
N, NF, NB, C, T = 3, 9, 27, 16, 128
INFO = 61


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


def sim(PX, CTpad, PERpad, order):
    PY = PX * N
    CT = PY * N + CTpad
    O_U, O_SX, O_SY, O_SZ, O_UX = 0, CT, 2 * CT, 3 * CT, 4 * CT
    PER = ((5 * CT + INFO) | 1) + PERpad
    idx3 = lambda i, j, k: i + PX * j + PY * k
    total = 0

    def split(it, X):
        if order == "cellfast":
            return it % C, it // C
        return it // X, it % X

    def run(nitems, fn):
        nonlocal total
        for w in range(T // 32):
            for rnd in range((nitems + T - 1) // T):
                insts = {}
                for lane in range(32):
                    it = rnd * T + w * 32 + lane
                    if it >= nitems:
                        continue
                    for key, a in fn(it):
                        insts.setdefault(key, []).append((lane, a))
                for ad in insts.values():
                    total += wav(ad)

    def A(it):
        cl, r = split(it, 3 * NF)
        d, tl = divmod(r, NF)
        p, q = tl % N, tl // N
        st = [1, PX, PY][d]
        b0 = [idx3(0, p, q), idx3(p, 0, q), idx3(p, q, 0)][d]
        base = cl * PER
        out = [(("Ar", l), base + O_U + b0 + l * st) for l in range(N)]
        out += [(("Aw", l), base + [O_SX, O_SY, O_SZ][d] + b0 + l * st) for l in range(N)]
        if d == 0:
            out += [(("Aux", i), base + O_UX + b0 + i) for i in range(N)]
        return out
    run(C * 3 * NF, A)

    def B(it):
        cl, tl = split(it, NF)
        b0 = idx3(0, tl % N, tl // N)
        base = cl * PER
        o = []
        for l in range(N):
            o += [(("Bra", l), base + O_SY + b0 + l), (("Brb", l), base + O_SZ + b0 + l),
                  (("Bwa", l), base + O_SY + b0 + l), (("Bwb", l), base + O_SZ + b0 + l)]
        return o
    run(C * NF, B)

    def Cs(it):
        cl, tl = split(it, NF)
        b0 = idx3(tl % N, 0, tl // N)
        base = cl * PER
        o = []
        for l in range(N):
            o += [(("C1", l), base + O_UX + b0 + l * PX), (("C2", l), base + O_SX + b0 + l * PX),
                  (("C3", l), base + O_SZ + b0 + l * PX), (("C4", l), base + O_SY + b0 + l * PX),
                  (("C5", l), base + O_SX + b0 + l * PX), (("C6", l), base + O_SZ + b0 + l * PX)]
        return o
    run(C * NF, Cs)

    def D(it):
        cl, tl = split(it, NF)
        b0 = idx3(tl % N, tl // N, 0)
        base = cl * PER
        o = []
        for l in range(N):
            o += [(("D1", l), base + O_SX + b0 + l * PY), (("D2", l), base + O_SZ + b0 + l * PY),
                  (("D3", l), base + O_U + b0 + l * PY)]
        return o
    run(C * NF, D)
    return total, PER


if __name__ == "__main__":
    print("round-1 (PX 3, cell-major):", sim(3, 0, 0, "cellmajor"))
    res = []
    for PX in (3, 4, 5):
        for CTpad in range(0, 8):
            for PERpad in range(0, 16):
                for order in ("cellmajor", "cellfast"):
                    t, per = sim(PX, CTpad, PERpad, order)
                    res.append((t, PX, CTpad, PERpad, order, per))
    res.sort()
    for r in res[:10]:
        print(r)
