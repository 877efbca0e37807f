"""3D sum-factorised Burgers operator on the B200 (reference ``semopt/ops.py`` with a
three-axis grid).

``SemOperator3D`` has the reference ``SemOperator`` surface for ``grid.dim == 3``
(apply_rhs / apply_jacobian / apply_jacobian_transpose on 3-component fields,
``counters``, ``max_matrix_dim``, ``densify``) and the launch interface the time loop
and the adjoint sweep drive (``launch_rk_stage``, ``launch_adj_stage``,
``launch_terminal``), so ``integrate``, ``sweep``, ``AssimilationProblem.evaluate``
and ``minimize`` run on 3D boxes unchanged.  Each apply is two kernels of
``libsemb200.so`` (element contraction, node gather: ``csrc/sem3d.cu``); stage
combinations are the library's vector kernels with the reference association order.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import NumericFailure, ValidationError
from .grid import Grid3D
from .ops import BURGERS, ComposedStages, _stream_handle, _torch, device_to_host, host_to_device


class _Plan3D:
    """Owns one sem3d_plan* (C ABI)."""

    def __init__(self, grid, nu, K3, Dw, T3):
        lib = _lib.load()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (np.stack(K3), Dw, np.stack(T3), grid.minv_pattern, grid.mass_pattern)]
        els = (ctypes.c_int64 * 3)(*[ax.elements for ax in grid.axes])
        handle = ctypes.c_void_p()
        rc = lib.sem3d_plan_create(els, grid.N, float(nu), *[a.ctypes.data for a in arrs],
                                   ctypes.byref(handle))
        if rc != 0:
            raise ValidationError(_lib.last_error())
        self.handle, self._lib = handle, lib
        self.ndof = lib.sem3d_plan_ndof(handle)
        self.work_size = lib.sem3d_work_size(handle)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.sem3d_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self.handle = None


class SemOperator3D(ComposedStages):
    """Matrix-free 3D Burgers operator bundle (ops.py:84-257 with dim 3)."""

    def __init__(self, grid, coef, device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("SemOperator3D needs a CUDA device (no CPU fallback)")
        if not isinstance(grid, Grid3D):
            raise ValidationError("SemOperator3D needs a 3D grid (grid_3d / build_grid with 3 axes)")
        if coef.advection != BURGERS:
            raise ValidationError("the B200 3D kernels implement Burgers advection")
        if grid.N > _lib.load().sem3d_max_degree():
            raise ValidationError(f"degree {grid.N} exceeds the 3D kernel limit "
                                  f"{_lib.load().sem3d_max_degree()}")
        self.grid, self.coef, self.batch = grid, coef, 1
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        b = grid.bases[0]
        w = b.weights
        self._dw = b.diff * w[:, None]                                   # ops.py:104
        self._kmat = []
        for ax in grid.axes:                                             # ops.py:105-106
            k = (2.0 / ax.element_length) * (b.diff.T * w) @ b.diff
            self._kmat.append(0.5 * (k + k.T))
        m1, m2, m3 = grid.mvec                                           # ops.py:109-115
        self._transverse = [m2[:, None] * m3[None, :], m1[:, None] * m3[None, :],
                            m1[:, None] * m2[None, :]]
        self.max_matrix_dim = grid.N + 1
        with _torch().cuda.device(self.device):   # the plan belongs to (and launches on) this device
            self._plan = _Plan3D(grid, coef.nu, self._kmat, self._dw, self._transverse)
        self.ndof = grid.nglobal
        self.shape = (self.ndof,)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._work = torch.empty(int(self._plan.work_size), dtype=torch.float64, device=self.device)
        self._J = torch.empty(1, dtype=torch.float64, device=self.device)
        self.counters = {"rhs": 0, "jac": 0, "jact": 0}
        self.last_sweep_stats = {}
        self._tmp = {}

    # -- plumbing (same contract as SemOperator) ----------------------------------

    def field(self, x, name="field"):
        torch = _torch()
        host = not isinstance(x, torch.Tensor)
        t = torch.as_tensor(np.asarray(x, dtype=np.float64) if host else x)
        if tuple(t.shape) != self.shape:
            raise ValidationError(f"{name} has shape {tuple(t.shape)}, expected {self.shape}")
        if t.dtype != torch.float64:
            raise ValidationError(f"{name} must be float64, got {t.dtype}")
        if t.device != self.device:
            t = host_to_device(t, self.device) if t.device.type == "cpu" else t.to(self.device)
        return t.contiguous(), host

    def empty(self):
        torch = _torch()
        return torch.empty(self.shape, dtype=torch.float64, device=self.device)

    def _stream(self):
        return _stream_handle(self.device)

    def flags(self, reset=True):
        v = int(self._flag.item())
        if v and reset:
            self._flag.zero_()
        return v

    def raise_for_flags(self, names=("state", "tangent")):
        v = self.flags()
        if v & _lib.SEM1D_FLAG_STATE_NONFINITE:
            raise NumericFailure(f"{names[0]} contains NaN/Inf")
        if v & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
            raise NumericFailure(f"{names[1]} contains NaN/Inf")
        return v

    @staticmethod
    def _isfinite_all(t):
        torch = _torch()
        return bool(torch.isfinite(t).all().item())

    def step_fused_supported(self):
        return False

    def rk_error_norm(self, u_new, u, k2, dt, cfg):
        """Embedded-pair weighted error (timeloop.py:205-210) -- the 1D operator's device
        reduction, which only needs ndof / device / stream."""
        from .ops import SemOperator
        return SemOperator.rk_error_norm(self, u_new, u, k2, dt, cfg)

    def _require_single(self, what):
        return None

    # -- raw launches ----------------------------------------------------------------

    def launch_rhs(self, u, out):
        _lib.check(_lib.load().sem3d_rhs(self._plan.handle, u.data_ptr(), out.data_ptr(),
                                         self._work.data_ptr(), self._flag.data_ptr(), self._stream()),
                   "sem3d_rhs")

    def launch_jac(self, u, v, out):
        _lib.check(_lib.load().sem3d_jac(self._plan.handle, u.data_ptr(), v.data_ptr(), out.data_ptr(),
                                         self._work.data_ptr(), self._flag.data_ptr(), self._stream()),
                   "sem3d_jac")

    def launch_jact(self, u, z, out):
        _lib.check(_lib.load().sem3d_jact(self._plan.handle, u.data_ptr(), z.data_ptr(), out.data_ptr(),
                                          self._work.data_ptr(), self._flag.data_ptr(), self._stream()),
                   "sem3d_jact")

    def launch_rk_stage(self, U_in, k_out, base, terms, coefs, dt, Y, check):
        """k = F(U_in), Y = base + dt * combination (sem1d_rk_stage semantics)."""
        self.compose_rk_stage(U_in, k_out, base, terms, coefs, dt, Y, check)

    def launch_adj_stage(self, U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out):
        """z = b lam + sum a_j l_j; l = dt J^T(U) z; lam_out = ((lam + L_0) + L_1) + ..."""
        self.compose_adj_stage(U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out)

    # -- Crank-Nicolson (sem3d_cn_*: the native Newton / GMRES drivers over the 3D applies) --

    def _cn_work(self, restart):
        torch = _torch()
        ws = getattr(self, "_cn_ws", None)
        if ws is None or ws[0] != int(restart):
            n = _lib.load().sem3d_cn_work_size(self._plan.handle, int(restart))
            if n < 0:
                raise ValidationError(f"gmres_restart={restart} outside the kernel limit 1..64")
            self._cn_ws = (int(restart), torch.zeros(int(n), dtype=torch.float64, device=self.device))
        return self._cn_ws[1]

    def launch_cn_step(self, u, v, dt, cfg, st):
        from .ops import SemOperator
        work = self._cn_work(cfg.gmres_restart)
        self._flag.zero_()
        p = SemOperator._cn_params(cfg)
        _lib.check(_lib.load().sem3d_cn_step(self._plan.handle, u.data_ptr(), v.data_ptr(), float(dt),
                                             ctypes.byref(p), work.data_ptr(), self._flag.data_ptr(),
                                             ctypes.byref(st), self._stream()), "sem3d_cn_step")

    def launch_cn_adjoint_step(self, u_n, u_np1, lam, lam_out, dt, cfg, st):
        from .ops import SemOperator
        work = self._cn_work(cfg.gmres_restart)
        self._flag.zero_()
        p = SemOperator._cn_params(cfg)
        _lib.check(_lib.load().sem3d_cn_adjoint_step(
            self._plan.handle, u_n.data_ptr(), u_np1.data_ptr(), lam.data_ptr(), lam_out.data_ptr(),
            float(dt), ctypes.byref(p), work.data_ptr(), self._flag.data_ptr(), ctypes.byref(st),
            self._stream()), "sem3d_cn_adjoint_step")

    def launch_terminal(self, uN, ud, lam, J_out):
        _lib.check(_lib.load().sem3d_terminal(self._plan.handle, uN.data_ptr(), ud.data_ptr(), lam.data_ptr(),
                                              J_out.data_ptr(), self._work.data_ptr(), self._stream()),
                   "sem3d_terminal")

    # -- reference surface -----------------------------------------------------------

    def _apply(self, launch, names, *xs):
        ts = [self.field(x, nm)[0] for x, nm in zip(xs, names)]
        host = not isinstance(xs[0], _torch().Tensor)
        out = self.empty()
        launch(*ts, out)
        self.raise_for_flags((names[0], names[-1]))
        return device_to_host(out) if host else out

    def apply_rhs(self, u):
        """f(u) = M^-1 gather(P_e(scatter(u))) (ops.py:232-236)."""
        self.counters["rhs"] += 1
        return self._apply(self.launch_rhs, ("state",), u)

    def apply_jacobian(self, u, w):
        self.counters["jac"] += 1
        return self._apply(self.launch_jac, ("state", "tangent"), u, w)

    def apply_jacobian_transpose(self, u, z):
        self.counters["jact"] += 1
        return self._apply(self.launch_jact, ("state", "cotangent"), u, z)

    def densify(self, u):
        """Dense J by columns (ops.py:259-273); verification only, n <= 5000."""
        n = self.grid.nglobal
        if n > 5000:
            raise ValidationError(f"densify refused: {n} unknowns exceeds limit 5000")
        torch = _torch()
        ut, _ = self.field(u, "state")
        cols = torch.empty((n, n), dtype=torch.float64, device=self.device)
        e = torch.zeros(n, dtype=torch.float64, device=self.device)
        out = self.empty()
        for k in range(n):
            e[k] = 1.0
            self.launch_jac(ut, e, out)
            cols[:, k] = out
            e[k] = 0.0
        self.counters["jac"] += n
        return cols.cpu().numpy()
