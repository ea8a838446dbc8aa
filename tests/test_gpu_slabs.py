"""z-slab decomposition on the device (paper_2107_07776_b200/slabs.py).

One GPU: the ranks are emulated one after another in one process -- no kernel waits on
another rank (B200_PROFILING.md) -- each with its own libdgb.so context on its local
layers (owned + ghost) and the fast kernels restricted to the owned cells
(dgb_set_cell_range).  The ghost layers are filled with exactly what the halo exchange
delivers (the neighbours' owned boundary layers).  Every rank's owned result must equal
the single-domain device apply; the multi-rank transport itself is covered on CPU
(tests/test_slabs.py, gloo).  Then a world-size-1 NCCL solve through the distributed
Krylov layer against the reference's cg_solve / gmres_solve."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = 2.0 - 2.0 ** 0.5


@pytest.mark.parametrize("n,ku,world", [(6, 3, 2), (7, 2, 3), (5, 4, 2), (8, 2, 4)])
def test_emulated_ranks_match_single_domain_apply(gpu, n, ku, world):
    import torch
    from paper_2107_07776_b200 import slabs
    D = gpu.DGContext(3, n, ku, ku - 1)
    w = torch.from_numpy(gpu.seeded_uniform(1, D.n_u)).cuda()
    x = torch.from_numpy(gpu.seeded_uniform(2, D.n_u)).cuda()
    xp = torch.from_numpy(gpu.seeded_uniform(3, D.n_p)).cuda()
    coefs = (1.0 / (G * 1e-3), 0.005, 0.5, 0.0)
    y, yp = D.zeros(), D.zeros(gpu.SPACE_P)
    gpu.apply_momentum(D, gpu.MomentumCtx(*coefs, advecting=w), x, y)
    gpu.apply_pressure_helmholtz(D, 2.3, xp, yp)
    for r in range(world):
        part = slabs.SlabPartition(n, world, r)
        be = slabs.DeviceSlabBackend(part, ku, ku - 1)
        assert be.ctx.fast_path_active
        nu, npb = be.nbc_u, be.nbc_p
        lo, hi = part.g0 * n * n, part.g1 * n * n   # local cells = owned + ghosts (halo-filled)
        ly, lyp = be.zeros(be.n_u), be.zeros(be.n_p)
        be.momentum(coefs, w[lo * nu:hi * nu].clone(), x[lo * nu:hi * nu].clone(), ly)
        be.pressure(2.3, xp[lo * npb:hi * npb].clone(), lyp)
        c0, c1 = part.global_cells
        ou, op = part.owned(nu), part.owned(npb)
        assert float((ly[ou] - y[c0 * nu:c1 * nu]).norm() / y[c0 * nu:c1 * nu].norm()) <= 1e-14
        assert float((lyp[op] - yp[c0 * npb:c1 * npb]).norm() / yp[c0 * npb:c1 * npb].norm()) <= 1e-14
        # only the owned cells were computed: the ghost rows are untouched (still zero);
        # the axis-aligned fast momentum kernel covers K <= 3 (K = 4 runs the generic
        # kernel, which computes every local cell -- same owned result)
        gp = float(lyp[:op.start].abs().sum() + lyp[op.stop:].abs().sum())
        gu = float(ly[:ou.start].abs().sum() + ly[ou.stop:].abs().sum())
        assert gp == 0.0 and (gu == 0.0 or ku == 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_distributed_krylov_world1_nccl_matches_reference(ref, gpu):
    import torch
    import torch.distributed as tdist
    from paper_2107_07776_b200 import slabs
    n, ku = 4, 2
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        part = slabs.SlabPartition(n, 1, 0)
        be = slabs.DeviceSlabBackend(part, ku, ku - 1)
        comm = slabs.TorchComm()
        R = ref.RefCtx(3, n, ku, ku - 1)
        w, bu, bp = ref.seeded_uniform(1, R.n_u), ref.seeded_uniform(5, R.n_u), ref.seeded_uniform(4, R.n_p)
        coefs = (1.0 / (G * 1e-3), 0.005, 0.5, 0.0)
        A = slabs.DistOperator(be, comm, "momentum", coefs=coefs, w=torch.from_numpy(w).cuda())
        Ap = slabs.DistOperator(be, comm, "pressure", mass_coef=2.3)
        xp = be.zeros(be.n_p)
        rp = slabs.cg_solve(Ap, torch.from_numpy(bp).cuda(), xp, inv=slabs.jacobi_inverse(Ap, Ap.diagonal()))
        xu = be.zeros(be.n_u)
        ru = slabs.gmres_solve(A, torch.from_numpy(bu).cuda(), xu, restart=20,
                               inv=slabs.jacobi_inverse(A, A.diagonal()))
        xr, itr, _ = R.solve(1, 0, (2.3, 0, 0, 0), None, bp, np.zeros(R.n_p))
        xg, itg, _ = R.solve(0, 1, coefs, w, bu, np.zeros(R.n_u), restart=20)
        assert abs(rp.iterations - itr) <= 1 and abs(ru.iterations - itg) <= 1, (rp, itr, ru, itg)
        rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel(xp.cpu().numpy(), xr) <= 1e-8 and rel(xu.cpu().numpy(), xg) <= 1e-8
    finally:
        tdist.destroy_process_group()
