"""CPU test double of the rank-local operator for the multi-process (gloo) tests of
dist.py: the same launch interface as SemOperator, computed by the oracle.  Test
infrastructure only -- it lets the partition / ghost-exchange / engine logic run on
CPU ranks; the GPU kernels themselves are covered by the -m gpu tests."""

import numpy as np
import torch

from oracle import semref as R


class CpuLocalOp:
    def __init__(self, grid, coef):
        ax = grid.axis
        mesh = R.Mesh1D(ax.xa, ax.xb, ax.elements, ax.degree, grid.periodic)
        mesh.h = grid.h                           # the shard uses the global h exactly
        mesh.mass = mesh.assemble(np.broadcast_to((mesh.h / 2.0) * mesh.rho,
                                                  (ax.elements, ax.degree + 1)))
        self.ref = R.BurgersOracle(mesh, coef.nu)
        self.grid, self.coef = grid, coef
        self.device = torch.device("cpu")
        self.batch = 1
        self.counters = {"rhs": 0, "jac": 0, "jact": 0}
        self.max_matrix_dim = ax.degree + 1

    @staticmethod
    def _np(t):
        return t.detach().cpu().numpy()

    def flags(self, reset=True):
        return 0

    def launch_rhs(self, u, out):
        out.copy_(torch.from_numpy(self.ref.rhs(self._np(u))))

    def launch_jac(self, u, v, out):
        out.copy_(torch.from_numpy(self.ref.jac(self._np(u), self._np(v))))

    def launch_jact(self, u, z, out):
        out.copy_(torch.from_numpy(self.ref.jact(self._np(u), self._np(z))))

    def launch_rk_stage(self, U_in, k_out, base, terms, coefs, dt, Y, check):
        k = self.ref.rhs(self._np(U_in))
        if k_out is not None:
            k_out.copy_(torch.from_numpy(k))
        vals = [k if t is None else self._np(t) for t in terms]
        b = self._np(base)
        if len(vals) == 1:
            y = b + (dt * coefs[0]) * vals[0]
        else:
            s = coefs[0] * vals[0]
            for c, v in zip(coefs[1:], vals[1:]):
                s = s + c * v
            y = b + dt * s
        Y.copy_(torch.from_numpy(y))

    def launch_adj_stage(self, U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out):
        lm = self._np(lam)
        z = b * lm
        for t, a in zip(l_terms, a_coefs):
            z = z + a * self._np(t)
        l = dt * self.ref.jact(self._np(U), z)
        if l_out is not None:
            l_out.copy_(torch.from_numpy(l))
        if lam_out is not None:
            acc = lm
            for t in acc_terms:
                acc = acc + (l if t is None else self._np(t))
            lam_out.copy_(torch.from_numpy(acc))
