"""Multi-rank z-slab decomposition (paper_2107_07776_b200/slabs.py) on CPU:
gloo, world_size 2 and 3, the reference standing in for the local device operator
(tests/slab_oracle.py).  Parity against the single-domain reference: distributed applies
<= 1e-12 relative L2 on every owned DoF, distributed CG / GMRES (the reference's
algorithms, one halo exchange per apply, one all-reduce per dot) iteration counts +-1 and
solutions within the solver tolerance."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
G = 2.0 - 2.0 ** 0.5


def test_partition_covers_the_mesh_once():
    from paper_2107_07776_b200.slabs import SlabPartition
    for n, world in ((5, 1), (5, 2), (6, 4), (7, 3), (8, 8)):
        parts = [SlabPartition(n, world, r) for r in range(world)]
        cover = []
        for p in parts:
            cover += list(range(*p.global_cells))
            assert p.own1 - p.own0 == p.global_cells[1] - p.global_cells[0]
            assert p.ncells == (p.g1 - p.g0) * n * n
        assert cover == list(range(n ** 3))
        nbc = 5
        for p in parts:  # what a rank sends is exactly what its peer receives (same global cells)
            for peer, s, r in p.halo_plan(nbc):
                q = parts[peer]
                back = [rr for pp, ss, rr in q.halo_plan(nbc) if pp == p.rank][0]
                g_send = (p.g0 * n * n * nbc + s.start, p.g0 * n * n * nbc + s.stop)
                g_recv = (q.g0 * n * n * nbc + back.start, q.g0 * n * n * nbc + back.stop)
                assert g_send == g_recv and s.stop - s.start == n * n * nbc


def test_local_mesh_cells_are_the_global_cells(ref):
    from paper_2107_07776_b200.slabs import SlabPartition
    import slab_oracle
    n = 5
    full = ref.RefCtx(3, n, 2, 1)
    xf = full.cell_vertices()
    for world in (2, 3):
        for r in range(world):
            p = SlabPartition(n, world, r)
            be = slab_oracle.OracleSlabBackend(p, 2, 1)
            xl = be.R.cell_vertices()
            assert np.array_equal(xl, xf[p.g0 * n * n:p.g1 * n * n])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, n, ku, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, TESTS)
    import torch
    import torch.distributed as tdist
    import reforacle as ref
    import slab_oracle
    from paper_2107_07776_b200 import slabs
    tdist.init_process_group("gloo", init_method="env://", rank=rank, world_size=ws)
    try:
        part = slabs.SlabPartition(n, ws, rank)
        be = slab_oracle.OracleSlabBackend(part, ku, ku - 1)
        comm = slabs.TorchComm()
        c0, c1 = part.global_cells
        nu, npb = be.nbc_u, be.nbc_p
        gu = lambda seed: torch.from_numpy(ref.seeded_uniform(seed, n ** 3 * nu))
        gp = lambda seed: torch.from_numpy(ref.seeded_uniform(seed, n ** 3 * npb))

        def local(g, nbc):  # this rank's owned part of a global vector, ghosts left at zero
            x = be.zeros((part.g1 - part.g0) * n * n * nbc)
            x[part.owned(nbc)] = g[c0 * nbc:c1 * nbc]
            return x
        w = local(gu(1), nu)
        coefs = (1.0 / (G * 1e-3), 0.005, 0.5, 0.0)
        A = slabs.DistOperator(be, comm, "momentum", coefs=coefs, w=w)
        y = be.zeros(be.n_u)
        A.apply(local(gu(2), nu), y)
        Ap = slabs.DistOperator(be, comm, "pressure", mass_coef=2.3)
        yp = be.zeros(be.n_p)
        Ap.apply(local(gp(3), npb), yp)
        # Jacobi-CG on the pressure Helmholtz operator, Jacobi-GMRES on the momentum operator
        bp = local(gp(4), npb)
        xp = be.zeros(be.n_p)
        rp = slabs.cg_solve(Ap, bp, xp, rel_tol=1e-10, inv=slabs.jacobi_inverse(Ap, Ap.diagonal()))
        bu = local(gu(5), nu)
        xu = be.zeros(be.n_u)
        ru = slabs.gmres_solve(A, bu, xu, rel_tol=1e-10, restart=20, inv=slabs.jacobi_inverse(A, A.diagonal()))
        own_u, own_p = part.owned(nu), part.owned(npb)
        q.put((rank, c0, c1, y[own_u].numpy().copy(), yp[own_p].numpy().copy(), rp.iterations,
               xp[own_p].numpy().copy(), ru.iterations, xu[own_u].numpy().copy()))
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("ws,n,ku", [(2, 4, 2), (3, 5, 2), (2, 4, 3)])
def test_distributed_applies_and_solves_match_reference_gloo(ref, ws, n, ku):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, n, ku, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=280) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    R = ref.RefCtx(3, n, ku, ku - 1)
    nu, npb = 3 * (ku + 1) ** 3, ku ** 3
    w, x, xp = ref.seeded_uniform(1, R.n_u), ref.seeded_uniform(2, R.n_u), ref.seeded_uniform(3, R.n_p)
    coefs = (1.0 / (G * 1e-3), 0.005, 0.5, 0.0)
    want_u, want_p = R.momentum(coefs, w, x), R.pressure(2.3, xp)
    got_u = np.concatenate([r[3] for r in res])
    got_p = np.concatenate([r[4] for r in res])
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(got_u, want_u) <= 1e-12 and rel(got_p, want_p) <= 1e-12
    bp, bu = ref.seeded_uniform(4, R.n_p), ref.seeded_uniform(5, R.n_u)
    xr, itr, _ = R.solve(1, 0, (2.3, 0, 0, 0), None, bp, np.zeros(R.n_p), rel_tol=1e-10)
    assert all(abs(r[5] - itr) <= 1 for r in res), ([r[5] for r in res], itr)
    assert rel(np.concatenate([r[6] for r in res]), xr) <= 1e-8
    xg, itg, _ = R.solve(0, 1, coefs, w, bu, np.zeros(R.n_u), rel_tol=1e-10, restart=20)
    assert all(abs(r[7] - itg) <= 1 for r in res), ([r[7] for r in res], itg)
    assert rel(np.concatenate([r[8] for r in res]), xg) <= 1e-8
