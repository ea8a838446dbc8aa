"""Multi-GPU z-slab decomposition of the DG operators and Krylov solves (SURVEY 8(e),
8(f) item 4).

One process per GPU.  The n_el^3 Cartesian mesh is cut into contiguous z-slabs (cells are
numbered x fastest, z slowest -- mesh.cpp:590-608 -- so every z-layer of cells, and so
every layer of DoFs, is one contiguous block).  Each rank builds a local context on its
owned layers plus one ghost layer on each side that has a neighbour rank.  The operators
are element-centric (each cell integrates all of its faces, reading the neighbour's data),
so an owned cell's result is exact once its ghost neighbours hold current input values:

* per operator apply: ONE halo exchange of the input field -- the first / last owned layer
  goes to the lower / upper neighbour's ghost layer (contiguous slices, sent in place: no
  packing).  The momentum operator's advecting field is exchanged once per solve (it is
  constant inside GMRES).
* per Krylov dot / norm: ONE all-reduce of an 8-byte partial sum over the owned DoFs.

The solvers are the reference's (krylov.cpp:43-207: PCG with outer true-residual restarts,
right-preconditioned restarted GMRES with sequential modified Gram-Schmidt and Givens), so
a distributed solve reproduces the single-domain iteration counts up to the summation
order of the dots.

The local operator is a backend object (``DeviceSlabBackend``: this package's libdgb.so on
the rank's GPU, the fast kernels restricted to the owned cells); the halo / all-reduce
transport is ``TorchComm`` (torch.distributed: NCCL on GPUs, gloo on CPUs).  Nothing
here falls back to a CPU implementation: the device backend fails loudly without libdgb.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------
class SlabPartition:
    """z-slabs of generate_cartesian<3>(n_el, 0, 1) (mesh.cpp:572-615) over `world` ranks.

    Rank r owns global z-layers [z0, z1) (a near-even split); its local mesh holds layers
    [g0, g1) = the owned layers plus one ghost layer below / above when a neighbour rank
    exists.  Local cell c <-> global cell g0 * n^2 + c."""

    def __init__(self, n_el: int, world: int, rank: int):
        if not (1 <= world <= n_el) or not (0 <= rank < world):
            raise ValueError(f"slab partition: need 1 <= world ({world}) <= n_el ({n_el}), 0 <= rank < world")
        self.n, self.world, self.rank = n_el, world, rank
        base, rem = divmod(n_el, world)
        self.z0 = rank * base + min(rank, rem)
        self.z1 = self.z0 + base + (1 if rank < rem else 0)
        self.g0 = max(self.z0 - 1, 0)
        self.g1 = min(self.z1 + 1, n_el)
        self.layer = n_el * n_el
        self.ncells = (self.g1 - self.g0) * self.layer
        self.own0 = (self.z0 - self.g0) * self.layer      # owned local cells [own0, own1)
        self.own1 = self.own0 + (self.z1 - self.z0) * self.layer
        self.lower = rank - 1 if self.z0 > 0 else None
        self.upper = rank + 1 if self.z1 < n_el else None

    @property
    def global_cells(self) -> Tuple[int, int]:
        """Global cell range [c0, c1) owned by this rank."""
        return self.z0 * self.layer, self.z1 * self.layer

    def owned(self, nbc: int) -> slice:
        """Local DoF slice of the owned cells (nbc DoFs per cell)."""
        return slice(self.own0 * nbc, self.own1 * nbc)

    def halo_plan(self, nbc: int) -> List[Tuple[int, slice, slice]]:
        """(peer, send slice, receive slice) per neighbour: the owned boundary layer goes
        to the peer's ghost layer, the peer's owned boundary layer fills ours."""
        L = self.layer * nbc
        plan = []
        if self.lower is not None:  # ghost layer = local layer 0, first owned = local layer 1
            plan.append((self.lower, slice(self.own0 * nbc, self.own0 * nbc + L), slice(0, L)))
        if self.upper is not None:  # last owned layer, ghost = local layer after the owned ones
            plan.append((self.upper, slice(self.own1 * nbc - L, self.own1 * nbc), slice(self.own1 * nbc, self.own1 * nbc + L)))
        return plan

    def mesh_arrays(self):
        """(vertices, cell vertices, boundary ids) of the local layers [g0, g1), with the
        global vertex coordinates lo + (hi - lo) * id / n (mesh.cpp:587) so every cell is
        bit-identical to its global twin.  Global boundary faces keep their ids (2a / 2a+1,
        mesh.cpp:609-612); the outer z-faces of ghost layers get ids 4 / 5 too -- they
        belong to ghost cells only, whose results are never used."""
        n, nz = self.n, self.g1 - self.g0
        nx = n + 1
        k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(nx), np.arange(nx), indexing="ij")
        verts = np.stack([(1.0 - 0.0) * i.ravel() / n, (1.0 - 0.0) * j.ravel() / n,
                          (1.0 - 0.0) * (self.g0 + k.ravel()) / n], axis=1) + 0.0
        ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(n), np.arange(n), indexing="ij")
        ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
        cells = np.stack([((ck + ((b >> 2) & 1)) * nx + cj + ((b >> 1) & 1)) * nx + ci + (b & 1) for b in range(8)],
                         axis=1).astype(np.int32)
        bids = -np.ones((len(ci), 6), dtype=np.int32)
        for a, (co, lim) in enumerate(((ci, n), (cj, n), (ck, nz))):
            bids[co == 0, 2 * a] = 2 * a
            bids[co == lim - 1, 2 * a + 1] = 2 * a + 1
        return np.ascontiguousarray(verts, dtype=np.float64), cells, bids


# ---------------------------------------------------------------------------
# transport
# ---------------------------------------------------------------------------
class TorchComm:
    """Halo exchange (point-to-point, in place on the field's own storage) and 8-byte
    all-reduces over torch.distributed -- NCCL between GPUs, gloo on CPUs."""

    def __init__(self, group=None):
        import torch.distributed as tdist
        self.td = tdist
        self.group = group

    def halo(self, part: SlabPartition, x, nbc: int) -> None:
        ops = []
        for peer, s, r in part.halo_plan(nbc):
            ops.append(self.td.P2POp(self.td.isend, x[s], peer, self.group))
            ops.append(self.td.P2POp(self.td.irecv, x[r], peer, self.group))
        if ops:
            for req in self.td.batch_isend_irecv(ops):
                req.wait()

    def allreduce(self, v: float, like) -> float:
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=getattr(like, "device", "cpu"))
        self.td.all_reduce(t, group=self.group)
        return float(t.item())


# ---------------------------------------------------------------------------
# local operators on the device
# ---------------------------------------------------------------------------
class DeviceSlabBackend:
    """The rank's local operators: a libdgb.so context on the local layers (owned + ghost)
    whose fast kernels compute only the owned cells (dgb_set_cell_range)."""

    def __init__(self, part: SlabPartition, ku: int, kp: int, device: int = 0):
        from . import DGContext, SPACE_P, lib, _check
        self.part = part
        self.ctx = DGContext(3, part.n, ku, kp, device=device, mesh_arrays=part.mesh_arrays())
        _check(lib().dgb_set_cell_range(self.ctx.handle, part.own0, part.own1))
        self.nbc_u, self.nbc_p = 3 * (ku + 1) ** 3, (kp + 1) ** 3
        self.n_u, self.n_p = self.ctx.n_u, self.ctx.n_p
        self._space_p = SPACE_P

    def zeros(self, n: int):
        import torch
        return torch.zeros(n, dtype=torch.float64, device=f"cuda:{self.ctx.device}")

    def copy(self, x):
        return x.clone()

    def dot(self, x, y, nbc: int) -> float:
        s = self.part.owned(nbc)
        return float((x[s] * y[s]).sum())

    def momentum(self, coefs, w, x, y) -> None:
        from . import MomentumCtx, apply_momentum
        apply_momentum(self.ctx, MomentumCtx(*coefs, advecting=w), x, y)

    def momentum_diag(self, coefs, w, d) -> None:
        from . import MomentumCtx, momentum_diagonal
        momentum_diagonal(self.ctx, MomentumCtx(*coefs, advecting=w), d)

    def pressure(self, mc, x, y) -> None:
        from . import apply_pressure_helmholtz
        apply_pressure_helmholtz(self.ctx, mc, x, y)

    def pressure_diag(self, mc, d) -> None:
        from . import helmholtz_diagonal
        helmholtz_diagonal(self.ctx, mc, d)


# ---------------------------------------------------------------------------
# distributed operators + the reference's Krylov solvers
# ---------------------------------------------------------------------------
@dataclass
class DistResult:
    iterations: int
    residual: float


class DistSolverError(RuntimeError):
    def __init__(self, msg: str, history):
        super().__init__(msg)
        self.history = list(history)


class DistOperator:
    """A distributed square operator: y = A x on the owned DoFs (ghost entries of y are
    not meaningful).  kind: "momentum" (coefs, w) or "pressure" (mass_coef)."""

    def __init__(self, be, comm, kind: str, coefs=None, w=None, mass_coef: float = 0.0):
        self.be, self.comm, self.kind = be, comm, kind
        self.coefs, self.w, self.mc = coefs, w, mass_coef
        self.nbc = be.nbc_u if kind == "momentum" else be.nbc_p
        self.n = be.n_u if kind == "momentum" else be.n_p
        if kind == "momentum" and w is not None:
            comm.halo(be.part, w, self.nbc)  # constant for the whole solve: one exchange

    def apply(self, x, y) -> None:
        self.comm.halo(self.be.part, x, self.nbc)  # the one exchange per apply
        if self.kind == "momentum":
            self.be.momentum(self.coefs, self.w, x, y)
        else:
            self.be.pressure(self.mc, x, y)

    def diagonal(self):
        d = self.be.zeros(self.n)
        if self.kind == "momentum":
            self.be.momentum_diag(self.coefs, self.w, d)
        else:
            self.be.pressure_diag(self.mc, d)
        return d

    # collectives over the owned DoFs
    def dot(self, x, y) -> float:
        return self.comm.allreduce(self.be.dot(x, y, self.nbc), x)

    def norm(self, x) -> float:
        return math.sqrt(self.dot(x, x))


def jacobi_inverse(A: DistOperator, diag):
    """JacobiPreconditioner (krylov.cpp:27-41) over the owned DoFs; raises naming the first
    (global) dof with a zero diagonal.  Ghost entries of the inverse are 0."""
    s = A.be.part.owned(A.nbc)
    own = diag[s]
    idx = (own == 0).nonzero()
    if idx.numel():
        bad = int(idx[0, 0]) if idx.dim() > 1 else int(idx[0])
        raise DistSolverError(f"jacobi preconditioner: zero diagonal at dof "
                              f"{A.be.part.global_cells[0] * A.nbc + bad}", [])
    inv = A.be.zeros(A.n)
    inv[s] = 1.0 / own
    return inv


def cg_solve(A: DistOperator, b, x, rel_tol: float = 1e-10, abs_tol: float = 0.0, max_iter: int = 10000,
             inv=None) -> DistResult:
    """cg_solve (krylov.cpp:43-101) with distributed applies and dots."""
    be = A.be
    bnorm = A.norm(b)
    if bnorm == 0.0:
        x[:] = 0.0
        return DistResult(0, 0.0)
    tol = max(rel_tol * bnorm, abs_tol)
    r, z, p, q = be.zeros(A.n), be.zeros(A.n), be.zeros(A.n), be.zeros(A.n)
    hist, it = [], 0
    while True:
        A.apply(x, q)
        r[:] = b - q
        rnorm = A.norm(r)
        if rnorm <= tol:
            return DistResult(it, rnorm)
        if it >= max_iter:
            raise DistSolverError(f"cg: no convergence in {max_iter} iterations (residual {rnorm})", hist)
        rho_old, first = 0.0, True
        while it < max_iter:
            z[:] = r * inv if inv is not None else r
            rho = A.dot(r, z)
            if rho == 0.0:
                raise DistSolverError("cg: breakdown, <r,z> = 0", hist)
            if first:
                p[:] = z
                first = False
            else:
                p[:] = z + (rho / rho_old) * p
            rho_old = rho
            A.apply(p, q)
            pq = A.dot(p, q)
            if pq <= 0.0:
                raise DistSolverError("cg: operator not positive definite, <p,Ap> <= 0", hist)
            alpha = rho / pq
            x += alpha * p
            r -= alpha * q
            it += 1
            rnorm = A.norm(r)
            hist.append(rnorm)
            if rnorm <= tol:
                break


def gmres_solve(A: DistOperator, b, x, rel_tol: float = 1e-10, abs_tol: float = 0.0, max_iter: int = 10000,
                restart: int = 50, inv=None) -> DistResult:
    """gmres_solve (krylov.cpp:103-207): right-preconditioned restarted GMRES, sequential
    modified Gram-Schmidt (one all-reduce per projection), Givens on the host."""
    be = A.be
    bnorm = A.norm(b)
    if bnorm == 0.0:
        x[:] = 0.0
        return DistResult(0, 0.0)
    tol = max(rel_tol * bnorm, abs_tol)
    m = max(1, restart)
    V: list = []
    z, w, r = be.zeros(A.n), be.zeros(A.n), be.zeros(A.n)
    hist, it = [], 0
    while True:
        A.apply(x, w)
        r[:] = b - w
        beta = A.norm(r)
        if beta <= tol:
            return DistResult(it, beta)
        if it >= max_iter:
            raise DistSolverError(f"gmres: no convergence in {max_iter} iterations (residual {beta})", hist)
        if not V:
            V.append(be.zeros(A.n))
        V[0][:] = r * (1.0 / beta)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        while k < m and it < max_iter:
            z[:] = V[k] * inv if inv is not None else V[k]
            A.apply(z, w)
            it += 1
            for i in range(k + 1):
                h = A.dot(w, V[i])
                H[i, k] = h
                w -= h * V[i]
            hk1 = A.norm(w)
            H[k + 1, k] = hk1
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            denom = math.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = (1.0, 0.0) if denom == 0.0 else (H[k, k] / denom, H[k + 1, k] / denom)
            H[k, k], H[k + 1, k] = denom, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            res = abs(g[k + 1])
            hist.append(res)
            k += 1
            if res <= tol or hk1 == 0.0:
                break
            if k < m and len(V) <= k:
                V.append(be.zeros(A.n))
            if k < m:
                V[k][:] = w * (1.0 / hk1)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            t = g[i] - sum(H[i, j] * y[j] for j in range(i + 1, k))
            y[i] = t / H[i, i]
        w[:] = 0.0
        for j in range(k):
            w += y[j] * V[j]
        z[:] = w * inv if inv is not None else w
        x += z
