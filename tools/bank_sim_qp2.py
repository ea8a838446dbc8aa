"""Per-array layout search for the shared-memory work arrays of qp_sip_field
(fast_deformed.cuh), under the bank model of tools/bank_sim_sip1.py (64-bit accesses,
two half-warps, wavefronts = max distinct addresses per 8-byte bank slot).

Every shared instruction touches one array, so each array's layout is chosen on its own:
for every order of its dimensions (fastest first) and pads added to each stride, the
wavefronts of all its accesses (the stages' lane -> element maps, one instruction per
compile-time loop index) are summed.  Layouts are lexicographic with padded strides,
so they stay injective.  usage: python tools/bank_sim_qp2.py N Q"""
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


def ideal(addrs):
    return 1 if all(l < 16 for l, _ in addrs) or all(l >= 16 for l, _ in addrs) else 2


def arrays(N, Q):
    """name -> (dims {name: extent}, accesses [(items, lane -> {dim: value} except the
    per-instruction dims, per-instruction dims)])"""
    NF = N * N
    X = ({"qx": Q, "j": N, "k": N}, [
        (NF, lambda it: {"j": it % N, "k": it // N}, ["qx"]),        # C1 write, C5 read
        (NF, lambda it: {"j": it % N, "k": it // N}, ["qx"]),
        (Q * N, lambda it: {"qx": it // N, "k": it % N}, ["j"]),     # C2 read, C4 write
        (Q * N, lambda it: {"qx": it // N, "k": it % N}, ["j"])])
    Y = ({"qx": Q, "qy": Q, "k": N}, [
        (Q * N, lambda it: {"qx": it // N, "k": it % N}, ["qy"]),    # C2 write, C4 read
        (Q * N, lambda it: {"qx": it // N, "k": it % N}, ["qy"]),
        (Q * Q, lambda r: {"qx": r // Q, "qy": r % Q}, ["k"]),      # C3 read, write
        (Q * Q, lambda r: {"qx": r // Q, "qy": r % Q}, ["k"])])
    FL = ({"f": 6, "fld": 4, "p": N, "q": N}, [
        (6 * NF, lambda it: {"f": it // NF, "p": (it % NF) % N, "q": (it % NF) // N}, ["fld"]),  # F1 write
        (6 * N, lambda it: {"f": it // N, "q": it % N}, ["fld", "p"])])                          # F2 read
    FP = ({"f": 6, "fld": 6, "q": N, "qp": Q}, [
        (6 * N, lambda it: {"f": it // N, "q": it % N}, ["fld", "qp"]),   # F2 write
        (6 * Q, lambda it: {"f": it // Q, "qp": it % Q}, ["fld", "q"])])  # F3 read
    FA = ({"f": 6, "part": 3, "qp": Q, "b": N}, [
        (6 * Q, lambda it: {"f": it // Q, "qp": it % Q}, ["part", "b"]),  # F3 write
        (6 * N, lambda it: {"f": it // N, "b": it % N}, ["part", "qp"])])  # F4 read
    FO = ({"f": 6, "h": 2, "bp": N, "bq": N}, [
        (6 * N, lambda it: {"f": it // N, "bq": it % N}, ["h", "bp"])] +   # F4 write
        [(NF, (lambda a, s: lambda tn: {"f": 2 * a + s, "h": 1 - s * 0, "bp": tn % N, "bq": tn // N})(a, s), ["_"])
         for a in range(3) for s in range(2)] +                             # F5 reads (normal part)
        [(NF, (lambda a, s: lambda tn: {"f": 2 * a + s, "h": 0, "bp": tn % N, "bq": tn // N})(a, s), ["_"])
         for a in range(3) for s in range(2)])
    return {"X": X, "Y": Y, "FL": FL, "FP": FP, "FA": FA, "FO": FO}


def cost(dims, accesses, order, pads):
    strides, s = {}, 1
    for d, pad in zip(order, pads):
        strides[d] = s
        s = s * dims[d] + pad
    size = s
    tot = idl = 0
    for nitems, lanemap, inst_dims in accesses:
        inst_dims = [d for d in inst_dims if d in dims]
        for rnd in range((nitems + 31) // 32):
            for combo in itertools.product(*[range(dims[d]) for d in inst_dims]):
                ad = []
                for lane in range(32):
                    it = lane + 32 * rnd
                    if it >= nitems:
                        continue
                    v = lanemap(it)
                    v.update(zip(inst_dims, combo))
                    ad.append((lane, sum(strides[d] * v[d] for d in dims)))
                tot += wav(ad)
                idl += ideal(ad)
    return tot, idl, size, strides


def search(N, Q):
    out = {}
    for name, (dims, acc) in arrays(N, Q).items():
        cur = None
        names = list(dims)
        best = None
        for order in itertools.permutations(names):
            for pads in itertools.product(range(0, 4), repeat=len(names) - 1):
                c = cost(dims, acc, order, list(pads) + [0])
                key = (c[0], c[2])
                if best is None or key < best[0]:
                    best = (key, order, pads, c)
        d0 = cost(dims, acc, _default_order(name), [0] * len(names))
        out[name] = (best, d0)
    return out


def _default_order(name):
    return {"X": ["j", "k", "qx"], "Y": ["k", "qy", "qx"], "FL": ["p", "q", "fld", "f"], "FP": ["qp", "q", "fld", "f"],
            "FA": ["b", "qp", "part", "f"], "FO": ["bp", "bq", "h", "f"]}[name]


if __name__ == "__main__":
    N, Q = int(sys.argv[1]), int(sys.argv[2])
    res = search(N, Q)
    tb = td = ti = 0
    for name, (best, d0) in res.items():
        (tot, size), order, pads, c = best
        print(f"{name:3s} round-1 {d0[0]:4d} (ideal {d0[1]}) size {d0[2]:4d} | best {tot:4d} size {size:4d} "
              f"order {order} pads {pads} strides {c[3]}")
        tb += tot
        td += d0[0]
        ti += d0[1]
    print(f"total round-1 {td}, best {tb}, ideal {ti}")
