"""Local operators of one slab rank computed by the unmodified reference (oracle/_ref) --
TEST INFRASTRUCTURE for the CPU (gloo) tests of paper_2107_07776_b200/slabs.py: the
partition / halo / all-reduce logic runs exactly as on GPUs, with the reference standing
in for libdgb.so as the local operator."""
import numpy as np
import torch

import reforacle as ref


class OracleSlabBackend:
    def __init__(self, part, ku, kp):
        verts, cells, bids = part.mesh_arrays()
        h = ref.lib().ref_create_from_arrays(3, len(verts), ref.P(verts), len(cells), cells.ctypes.data_as(ref._ip),
                                             bids.ctypes.data_as(ref._ip), ku, kp)
        assert h, ref.lib().ref_last_error().decode()
        self.R = ref.RefCtx(handle=h)
        self.part = part
        self.nbc_u, self.nbc_p = 3 * (ku + 1) ** 3, (kp + 1) ** 3
        self.n_u, self.n_p = self.R.n_u, self.R.n_p

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def copy(self, x):
        return x.clone()

    def dot(self, x, y, nbc):
        s = self.part.owned(nbc)
        return float((x[s] * y[s]).sum())

    def momentum(self, coefs, w, x, y):
        y.copy_(torch.from_numpy(self.R.momentum(coefs, w.numpy(), x.numpy())))

    def momentum_diag(self, coefs, w, d):
        d.copy_(torch.from_numpy(self.R.momentum_diag(coefs, w.numpy())))

    def pressure(self, mc, x, y):
        y.copy_(torch.from_numpy(self.R.pressure(mc, x.numpy())))

    def pressure_diag(self, mc, d):
        d.copy_(torch.from_numpy(self.R.helmholtz_diag(mc)))
