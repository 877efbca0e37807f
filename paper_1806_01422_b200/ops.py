"""Matrix-free Burgers operator on the B200 (reference ``semopt/ops.py``).

``SemOperator`` keeps the reference's duck-typed plugin surface
(``apply_rhs``, ``apply_jacobian``, ``apply_jacobian_transpose``, ``densify``,
``counters``, ``grid``, ``coef``, ``max_matrix_dim``; ops.py:84-273) but every
apply is ONE fused sm_100a kernel launched through the C ABI
(``include/sem1d.h``): scatter, the element contractions, the nonlinear and
viscous terms, the gather, M^-1 and the Dirichlet mask never leave the SM.

Fields are fp64 torch tensors on the operator's CUDA device.  numpy inputs
are accepted for drop-in use: they are copied to the device and the result is
copied back (that host round trip is what ``bench.py`` reports as ``e2e``).
There is no CPU fallback: without the library or a GPU the constructor raises.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib
from .errors import NumericFailure, ValidationError

BURGERS = "burgers"
LINEAR = "linear"
NONE = "none"

_DENSIFY_LIMIT = 5000


class PdeCoefficients:
    """Viscosity plus advection kind ('burgers' | 'linear' | 'none') (ops.py:42-60).
    Burgers runs the fused tensor-core kernels; 'linear' (constant speed) and 'none'
    run the generic 1D apply kernel with composed stages (sem1d_plan_set_advection)."""

    def __init__(self, nu, advection=BURGERS, speed=None):
        if not np.isfinite(nu) or nu < 0.0:
            raise ValidationError(f"viscosity must be >= 0, got {nu!r}")
        if advection not in (BURGERS, LINEAR, NONE):
            raise ValidationError(f"unknown advection kind {advection!r}")
        self.nu = float(nu)
        self.advection = advection
        if advection == LINEAR:
            if speed is None:
                raise ValidationError("linear advection needs a speed")
            self.speed = np.atleast_1d(np.asarray(speed, dtype=float))
        else:
            self.speed = None

    def __repr__(self):
        return f"PdeCoefficients(nu={self.nu}, advection={self.advection!r}, speed={self.speed})"


class ComposedStages:
    """RK and adjoint stages composed from the F / J^T applies and the library's vector
    kernels (sem1d_vec_*), with the association orders of sem1d_rk_stage /
    sem1d_adj_stage -- for operators without fused stage kernels (3D boxes, the
    linear / none advection kinds).  Needs launch_rhs / launch_jact, _buf, _flag, _stream."""

    def _numel(self):
        return self.ndof * self.batch

    def _buf(self, key):
        bufs = self.__dict__.setdefault("_tmp", {})
        t = bufs.get(key)
        if t is None:
            t = self.empty()
            bufs[key] = t
        return t

    def compose_rk_stage(self, U_in, k_out, base, terms, coefs, dt, Y, check):
        k = k_out if k_out is not None else self._buf("k")
        self.launch_rhs(U_in, k)
        ptrs = _lib.ptr_array([(k if t is None else t).data_ptr() for t in terms])
        _lib.check(_lib.load().sem1d_vec_rk_combine(
            self._numel(), base.data_ptr(), float(dt), len(terms), ptrs, _lib.dbl_array(coefs),
            Y.data_ptr(), 1 if check else 0, self._flag.data_ptr(), self._stream()), "sem1d_vec_rk_combine")

    def compose_adj_stage(self, U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out):
        lib, s, n = _lib.load(), self._stream(), self._numel()
        z, jt = self._buf("z"), self._buf("jt")
        _lib.check(lib.sem1d_vec_adj_combine(n, lam.data_ptr(), float(b), len(l_terms),
                                             _lib.ptr_array([t.data_ptr() for t in l_terms]),
                                             _lib.dbl_array(a_coefs), z.data_ptr(), s), "sem1d_vec_adj_combine")
        self.launch_jact(U, z, jt)
        lo = l_out if l_out is not None else self._buf("l")
        _lib.check(lib.sem1d_vec_scale(n, jt.data_ptr(), float(dt), lo.data_ptr(), s), "sem1d_vec_scale")
        if lam_out is not None:
            acc = [lo if t is None else t for t in (acc_terms or [])]
            _lib.check(lib.sem1d_vec_accumulate(n, lam.data_ptr(), len(acc),
                                                _lib.ptr_array([t.data_ptr() for t in acc]),
                                                lam_out.data_ptr(), s), "sem1d_vec_accumulate")


def _torch():
    import torch
    return torch


def _stream_handle(device):
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


# numpy fields on the drop-in path (a semopt user's apply_rhs(u) with u a numpy array).
# Pageable copies run at a few GB/s and the fresh result array page-faults on first touch,
# so large fields move through pinned memory instead: inputs stream through a ring of
# pinned chunks (the CPU copy of chunk k+1 overlaps the DMA of chunk k), results are read
# back into pinned arrays from torch's caching host allocator (reused once the caller drops
# them), handed to the caller as numpy views.
_STAGE_MIN_BYTES = 1 << 20
_STAGE_CHUNK = 1 << 21           # doubles per pinned chunk (16 MB)
_STAGE_SLOTS = 3


class _HostStaging:
    def __init__(self):
        self.bufs = None
        self.events = [None] * _STAGE_SLOTS
        self.lock = threading.Lock()      # one ring per process; callers may be concurrent

    def h2d(self, src, dst):
        """dst (device) <- src (pageable CPU tensor), on dst's current stream."""
        with self.lock:
            self._h2d(src, dst)

    def _h2d(self, src, dst):
        torch = _torch()
        if self.bufs is None:
            self.bufs = [torch.empty(_STAGE_CHUNK, dtype=torch.float64, pin_memory=True)
                         for _ in range(_STAGE_SLOTS)]
        s, d = src.reshape(-1), dst.reshape(-1)
        stream = torch.cuda.current_stream(dst.device)
        n = s.numel()
        for k, off in enumerate(range(0, n, _STAGE_CHUNK)):
            b = k % _STAGE_SLOTS
            if self.events[b] is not None:
                self.events[b].synchronize()          # the DMA out of this slot has drained
            m = min(_STAGE_CHUNK, n - off)
            buf = self.bufs[b][:m]
            buf.copy_(s[off:off + m])
            d[off:off + m].copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.events[b] = ev


_staging = _HostStaging()


def host_to_device(x, device):
    """A host field (numpy / CPU tensor) as a contiguous fp64 tensor on ``device``."""
    torch = _torch()
    t = torch.as_tensor(x).contiguous()
    if t.numel() * 8 < _STAGE_MIN_BYTES or t.dtype != torch.float64 or t.is_pinned():
        return t.to(device, non_blocking=False)
    out = torch.empty(t.shape, dtype=torch.float64, device=device)
    _staging.h2d(t, out)
    return out


def device_to_host(t):
    """A device result as a numpy array (pinned, read back in one DMA, for large fields)."""
    torch = _torch()
    if t.numel() * 8 < _STAGE_MIN_BYTES:
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


class _Plan:
    """Owns one sem1d_plan* (C ABI)."""

    def __init__(self, grid, nu, K, Dw, batch):
        lib = _lib.load()
        ax = grid.axis
        K = np.ascontiguousarray(K, dtype=np.float64)
        Dw = np.ascontiguousarray(Dw, dtype=np.float64)
        mp = np.ascontiguousarray(grid.mass_pattern, dtype=np.float64)
        mi = np.ascontiguousarray(grid.minv_pattern, dtype=np.float64)
        handle = _lib.c_void_p()
        rc = lib.sem1d_plan_create(ax.elements, ax.degree, 1 if grid.periodic else 0, float(nu),
                                   K.ctypes.data, Dw.ctypes.data, mp.ctypes.data, mi.ctypes.data,
                                   int(batch), _lib.ctypes.byref(handle))
        if rc != 0:
            msg = _lib.last_error()
            raise ValidationError(msg)
        self.handle = handle
        self._lib = lib
        self.ndof = lib.sem1d_plan_ndof(handle)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.sem1d_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self.handle = None


class SemOperator(ComposedStages):
    """Matrix-free SEM operator bundle for one (grid, coefficients) pair.

    ``batch`` > 1 makes every field a (batch, ndof) stack of independent
    problems sharing grid and viscosity (BASELINE config 4).
    """

    def __new__(cls, grid, coef, *args, **kwargs):
        # the reference's SemOperator serves 1D and 3D grids (ops.py:84-124): a 3D grid gets
        # the sum-factorised operator
        if cls is SemOperator and getattr(grid, "dim", 1) == 3:
            from .ops3d import SemOperator3D
            return SemOperator3D(grid, coef, device=kwargs.get("device", args[0] if args else None))
        return super().__new__(cls)

    def __init__(self, grid, coef, device=None, batch=1, sync_checks=True):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("SemOperator needs a CUDA device (the B200 path has no CPU fallback)")
        if grid.dim != 1:
            raise ValidationError("only 1D grids are supported on the B200 path")
        self.grid = grid
        self.coef = coef
        self.batch = int(batch)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        ax, b = grid.axis, grid.bases[0]
        w = b.weights
        # constants exactly as ops.py:103-107
        self._dw = b.diff * w[:, None]
        k = (2.0 / grid.h) * (b.diff.T * w) @ b.diff
        self._kmat = 0.5 * (k + k.T)
        self._minv = grid.minv_pattern
        self.max_matrix_dim = ax.degree + 1
        if ax.degree > _lib.load().sem1d_max_degree():
            raise ValidationError(f"degree {ax.degree} exceeds the kernel limit")
        with torch.cuda.device(self.device):   # the plan belongs to (and launches on) this device
            self._plan = _Plan(grid, coef.nu, self._kmat, self._dw, self.batch)
        self._adv = coef.advection != BURGERS
        if self._adv:
            if coef.advection == LINEAR and coef.speed.size != grid.ncomp:   # ops.py:95-100
                raise ValidationError(f"linear advection speed has {coef.speed.size} components, "
                                      f"grid has {grid.ncomp}")
            mode, a = (1, float(coef.speed[0])) if coef.advection == LINEAR else (2, 0.0)
            _lib.check(_lib.load().sem1d_plan_set_advection(self._plan.handle, mode, a),
                       "sem1d_plan_set_advection")
        self.ndof = grid.nglobal
        self.shape = (self.ndof,) if self.batch == 1 else (self.batch, self.ndof)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._work = torch.empty(max(1, _lib.load().sem1d_terminal_work_size(self._plan.handle)),
                                 dtype=torch.float64, device=self.device)
        self.counters = {"rhs": 0, "jac": 0, "jact": 0}
        self.sync_checks = sync_checks
        self.last_sweep_stats = {}

    # -- field plumbing -------------------------------------------------------

    def field(self, x, name="field"):
        """Validate and place an input; returns (tensor on device, came_from_host)."""
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
        """Read (and clear) the device non-finite flags -- one host sync."""
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

    @staticmethod
    def _out(t, host):
        return device_to_host(t) if host else t

    # -- raw launches (no validation, no sync): used by the engines -------------

    def launch_rhs(self, u, out):
        _lib.check(_lib.load().sem1d_rhs(self._plan.handle, u.data_ptr(), out.data_ptr(),
                                         self._flag.data_ptr(), self._stream()), "sem1d_rhs")

    def launch_jac(self, u, v, out):
        _lib.check(_lib.load().sem1d_jac(self._plan.handle, u.data_ptr(), v.data_ptr(),
                                         out.data_ptr(), self._flag.data_ptr(), self._stream()),
                   "sem1d_jac")

    def launch_jact(self, u, z, out):
        _lib.check(_lib.load().sem1d_jact(self._plan.handle, u.data_ptr(), z.data_ptr(),
                                          out.data_ptr(), self._flag.data_ptr(), self._stream()),
                   "sem1d_jact")

    def launch_rk_stage(self, U_in, k_out, base, terms, coefs, dt, Y, check):
        if self._adv:
            return self.compose_rk_stage(U_in, k_out, base, terms, coefs, dt, Y, check)
        ptrs = _lib.ptr_array([None if t is None else t.data_ptr() for t in terms])
        cf = _lib.dbl_array(coefs)
        _lib.check(_lib.load().sem1d_rk_stage(
            self._plan.handle, U_in.data_ptr(), None if k_out is None else k_out.data_ptr(),
            base.data_ptr(), len(terms), ptrs, cf, float(dt), Y.data_ptr(), 1 if check else 0,
            self._flag.data_ptr(), self._stream()), "sem1d_rk_stage")

    def launch_adj_stage(self, U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out):
        if self._adv:
            return self.compose_adj_stage(U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out)
        lp = _lib.ptr_array([t.data_ptr() for t in l_terms])
        ac = _lib.dbl_array(a_coefs)
        accp = _lib.ptr_array([None if t is None else t.data_ptr() for t in (acc_terms or [])])
        _lib.check(_lib.load().sem1d_adj_stage(
            self._plan.handle, U.data_ptr(), lam.data_ptr(), float(b), len(l_terms), lp, ac,
            float(dt), None if l_out is None else l_out.data_ptr(),
            len(acc_terms or []), accp, None if lam_out is None else lam_out.data_ptr(),
            self._flag.data_ptr(), self._stream()), "sem1d_adj_stage")

    def launch_terminal(self, uN, ud, lam, J_out):
        _lib.check(_lib.load().sem1d_terminal(self._plan.handle, uN.data_ptr(), ud.data_ptr(),
                                              lam.data_ptr(), J_out.data_ptr(),
                                              self._work.data_ptr(), self._stream()),
                   "sem1d_terminal")

    def launch_ens_forward(self, u0, traj, u_final, dts_dev, nsteps, scheme, flags):
        code = {"euler": 0, "rk3": 1, "rk4": 2}[scheme]
        _lib.check(_lib.load().sem1d_ens_forward(
            self._plan.handle, u0.data_ptr(), None if traj is None else traj.data_ptr(),
            u_final.data_ptr(), dts_dev.data_ptr(), int(nsteps), code, flags.data_ptr(),
            self._stream()), "sem1d_ens_forward")

    def launch_ens_adjoint(self, traj, lam_in, lam_out, dts_dev, nsteps, scheme, flags, check=True):
        """check=False: only lam_out is tested (SEM1D_FLAG_STEP_NONFINITE); a caller re-runs a
        flagged sweep with check=True to classify non-finite cotangents (sem1d_ens_adjoint_ex)."""
        code = {"euler": 0, "rk3": 1, "rk4": 2}[scheme]
        _lib.check(_lib.load().sem1d_ens_adjoint_ex(
            self._plan.handle, traj.data_ptr(), lam_in.data_ptr(), lam_out.data_ptr(),
            dts_dev.data_ptr(), int(nsteps), code, 1 if check else 0, flags.data_ptr(), self._stream()),
            "sem1d_ens_adjoint_ex")

    _SCHEME_CODES = {"euler": 0, "rk3": 1, "rk4": 2}

    def step_fused_supported(self):
        """Whole-step fused kernels apply (periodic batch-1 ring, n % 8 == 0, >= 2 tiles)."""
        if not hasattr(self, "_step_ok"):
            self._step_ok = bool(_lib.load().sem1d_step_supported(self._plan.handle)) and not self._adv
        return self._step_ok and getattr(self, "use_fused_steps", True)

    def launch_rk_step(self, u, u_new, dt, scheme, flag=None, tiles=None):
        """One fused step; ``flag``: device address of the int32 flag word to OR into
        (default the operator's own -- ``integrate`` passes per-step slots when it runs ahead,
        and then the step checks only its new state: a flagged step is re-run with the full
        classification before any exception is raised, sem1d_rk_step_ex).  ``tiles``:
        (first, count) ring tiles of the launch (N = 7; default all, see step_tiling)."""
        lo, cnt = tiles or (0, 0)
        _lib.check(_lib.load().sem1d_rk_step_ex(self._plan.handle, u.data_ptr(), u_new.data_ptr(), None,
                                                float(dt), self._SCHEME_CODES[scheme], 0 if flag else 1,
                                                int(lo), int(cnt), flag or self._flag.data_ptr(),
                                                self._stream()), "sem1d_rk_step_ex")

    def step_tiling(self, kind, stored, scheme):
        """(ntiles, owned elements per tile, ghost elements per side) of a whole-step launch
        (kind 0 forward, 1 adjoint): tile t reads elements [t*owned - ghost, (t+1)*owned + ghost)."""
        out = [_lib.ctypes.c_int() for _ in range(3)]
        _lib.check(_lib.load().sem1d_step_tiling(self._plan.handle, int(kind), 1 if stored else 0,
                                                 self._SCHEME_CODES[scheme], *[_lib.ctypes.byref(o) for o in out]),
                   "sem1d_step_tiling")
        return tuple(o.value for o in out)

    supports_flag_slots = True

    def flag_slots(self, k):
        """A zeroed device int32 array of (at least) k per-step flag words (cached)."""
        t = getattr(self, "_flag_slots_t", None)
        if t is None or t.numel() < k:
            t = _torch().zeros(k, dtype=_torch().int32, device=self.device)
            self._flag_slots_t = t
        return t

    def step_stages_supported(self):
        """The fused step pair that keeps the stage states in HBM applies (shared memory fits)."""
        if not hasattr(self, "_stages_ok"):
            self._stages_ok = bool(_lib.load().sem1d_step_stages_supported(self._plan.handle)) and not self._adv
        return self._stages_ok and self.step_fused_supported()

    def launch_rk_step_stages(self, u, u_new, stages, dt, scheme, flag=None, tiles=None):
        """One fused step that also writes the stage states U_1..U_{s-1} into `stages` (tiles
        as in launch_rk_step).  Always the classifying check: with the stage stores the
        outputs-only form measured slower (N = 7: 278 against 269 us on the config-2 field),
        and a classified flag is one the run-ahead's re-run would give anyway."""
        lo, cnt = tiles or (0, 0)
        _lib.check(_lib.load().sem1d_rk_step_ex(
            self._plan.handle, u.data_ptr(), u_new.data_ptr(), _lib.ptr_array([t.data_ptr() for t in stages]),
            float(dt), self._SCHEME_CODES[scheme], 1, int(lo), int(cnt),
            flag or self._flag.data_ptr(), self._stream()), "sem1d_rk_step_ex")

    def launch_adj_step_stages(self, u, stages, lam, lam_out, dt, scheme, flag=None, tiles=None):
        """One fused adjoint step reading the stored stage states (no recompute); checks as in
        launch_adj_step."""
        lo, cnt = tiles or (0, 0)
        _lib.check(_lib.load().sem1d_adj_step_ex(
            self._plan.handle, u.data_ptr(), _lib.ptr_array([t.data_ptr() for t in stages]), lam.data_ptr(),
            lam_out.data_ptr(), float(dt), self._SCHEME_CODES[scheme], 0 if flag else 1, int(lo), int(cnt),
            flag or self._flag.data_ptr(), self._stream()), "sem1d_adj_step_ex")

    def launch_adj_step(self, u, lam, lam_out, dt, scheme, flag=None, tiles=None):
        """One fused adjoint step; ``flag`` as in launch_rk_step: with a per-step flag word
        (``sweep`` running ahead) the step tests only its output lam_out and the sweep re-runs a
        flagged step with the classifying check (sem1d_adj_step_ex); ``tiles`` as in
        launch_rk_step."""
        lo, cnt = tiles or (0, 0)
        _lib.check(_lib.load().sem1d_adj_step_ex(self._plan.handle, u.data_ptr(), None, lam.data_ptr(),
                                                 lam_out.data_ptr(), float(dt), self._SCHEME_CODES[scheme],
                                                 0 if flag else 1, int(lo), int(cnt),
                                                 flag or self._flag.data_ptr(), self._stream()),
                   "sem1d_adj_step_ex")

    # -- implicit path (Crank-Nicolson) --------------------

    def _cn_work(self, restart):
        """Zero-initialised device workspace for sem1d_cn_* / sem1d_gmres (one per operator)."""
        torch = _torch()
        ws = getattr(self, "_cn_ws", None)
        if ws is None or ws[0] != int(restart):
            n = _lib.load().sem1d_cn_work_size(self._plan.handle, int(restart))
            if n < 0:
                raise ValidationError(f"gmres_restart={restart} outside the kernel limit 1..64")
            self._cn_ws = (int(restart), torch.zeros(int(n), dtype=torch.float64, device=self.device))
        return self._cn_ws[1]

    @staticmethod
    def _cn_params(cfg):
        return _lib.CnParams(float(cfg.newton_tol), int(cfg.newton_max), float(cfg.gmres_tol),
                             int(cfg.gmres_max), int(cfg.gmres_restart))

    def _require_single(self, what):
        if self.batch != 1:
            raise ValidationError(f"{what} needs a batch-1 operator")

    def launch_cn_step(self, u, v, dt, cfg, st):
        """v = Crank-Nicolson step of u (timeloop.py:154-186); accumulates into the CnStats st.
        Synchronises the stream at the reference's Newton / GMRES decision points."""
        import ctypes
        self._require_single("Crank-Nicolson")
        work = self._cn_work(cfg.gmres_restart)
        self._flag.zero_()
        p = self._cn_params(cfg)
        _lib.check(_lib.load().sem1d_cn_step(self._plan.handle, u.data_ptr(), v.data_ptr(), float(dt),
                                             ctypes.byref(p), work.data_ptr(), self._flag.data_ptr(),
                                             ctypes.byref(st), self._stream()), "sem1d_cn_step")

    def launch_cn_adjoint_step(self, u_n, u_np1, lam, lam_out, dt, cfg, st):
        """lam_out = transpose of the CN step map (adjoint.py:64-69)."""
        import ctypes
        self._require_single("Crank-Nicolson")
        work = self._cn_work(cfg.gmres_restart)
        self._flag.zero_()
        p = self._cn_params(cfg)
        _lib.check(_lib.load().sem1d_cn_adjoint_step(
            self._plan.handle, u_n.data_ptr(), u_np1.data_ptr(), lam.data_ptr(), lam_out.data_ptr(),
            float(dt), ctypes.byref(p), work.data_ptr(), self._flag.data_ptr(), ctypes.byref(st),
            self._stream()), "sem1d_cn_adjoint_step")

    def launch_gmres(self, p, alpha, b, x, cfg, st, transpose=False):
        """x = GMRES solution of (I + alpha J(p)) x = b (or J^T), scipy 1.18.1 semantics."""
        import ctypes
        self._require_single("GMRES")
        work = self._cn_work(cfg.gmres_restart)
        self._flag.zero_()
        prm = self._cn_params(cfg)
        _lib.check(_lib.load().sem1d_gmres(self._plan.handle, 1 if transpose else 0, p.data_ptr(),
                                           float(alpha), b.data_ptr(), x.data_ptr(), ctypes.byref(prm),
                                           work.data_ptr(), self._flag.data_ptr(), ctypes.byref(st),
                                           self._stream()), "sem1d_gmres")

    def rk_error_norm(self, u_new, u, k2, dt, cfg):
        """Weighted local truncation error of the embedded Kutta-3 pair
        (timeloop.py:205-210): mean sqrt(ratio) ("rms") or max ratio ("max").  One sync."""
        torch = _torch()
        self._require_single("adaptive stepping")
        if not hasattr(self, "_red"):
            self._red = torch.zeros(int(_lib.load().sem1d_reduce_work_size()) + 2,
                                    dtype=torch.float64, device=self.device)
        out = self._red[-1:]
        mx = cfg.wlte_form == "max"
        _lib.check(_lib.load().sem1d_rk_error_norm(
            self.ndof, u_new.data_ptr(), u.data_ptr(), k2.data_ptr(), float(dt), float(cfg.tol_a),
            float(cfg.tol_r), 1 if mx else 0, self._red.data_ptr(), out.data_ptr(), self._stream()),
            "sem1d_rk_error_norm")
        v = float(out.item())
        return v if mx else v / self.ndof

    # -- reference surface ------------------------------------------------------

    def apply_rhs(self, u):
        """f(u) = M^-1 gather(F_e(scatter(u))) (ops.py:232-236)."""
        ut, host = self.field(u, "state")
        self.counters["rhs"] += 1
        out = self.empty()
        self.launch_rhs(ut, out)
        if self.sync_checks:
            self.raise_for_flags(("state", "state"))
        return self._out(out, host)

    def apply_jacobian(self, u, w):
        """J(u) w (ops.py:238-244)."""
        ut, host = self.field(u, "state")
        wt, _ = self.field(w, "tangent")
        self.counters["jac"] += 1
        out = self.empty()
        self.launch_jac(ut, wt, out)
        if self.sync_checks:
            self.raise_for_flags(("state", "tangent"))
        return self._out(out, host)

    def apply_jacobian_transpose(self, u, z):
        """(M^-1 J)^T z = gather(J_e^T scatter(M^-1 z)) (ops.py:246-257)."""
        ut, host = self.field(u, "state")
        zt, _ = self.field(z, "cotangent")
        self.counters["jact"] += 1
        out = self.empty()
        self.launch_jact(ut, zt, out)
        if self.sync_checks:
            self.raise_for_flags(("state", "cotangent"))
        return self._out(out, host)

    def apply_host(self, u, v=None, w=None, kinds=None, chunks=8, out=None, slots=3):
        """F(u), J(u) v, J(u)^T w on HOST fields (pinned CPU tensors or numpy), streamed
        through the GPU in element chunks with copy/compute overlap (see HostStreamer).
        Returns a dict {"rhs", "jac", "jact"} of pinned CPU tensors (numpy for numpy
        input); ``out`` may supply some of them (float64 host tensors of the field's
        shape, pinned for overlap).  Raises NumericFailure like apply_* on non-finite
        input."""
        import torch
        if self.batch != 1:
            raise ValidationError("apply_host needs batch == 1")
        host_np = not isinstance(u, torch.Tensor)

        def prep(x, name):
            if x is None:
                return None
            t = torch.as_tensor(np.asarray(x, dtype=np.float64)) if not isinstance(x, torch.Tensor) else x
            if tuple(t.shape) != self.shape or t.dtype != torch.float64 or t.is_cuda:
                raise ValidationError(f"{name} must be a float64 host field of shape {self.shape}")
            return t
        u, v, w = prep(u, "state"), prep(v, "tangent"), prep(w, "cotangent")
        if kinds is None:
            kinds = ["rhs"] + (["jac"] if v is not None else []) + (["jact"] if w is not None else [])
        if out:
            for k, t in out.items():
                if (not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float64
                        or tuple(t.shape) != self.shape):
                    raise ValidationError(f"out[{k!r}] must be a float64 host tensor of shape {self.shape}")
        key = ("_streamer", chunks, slots)
        st = self.__dict__.get(key)
        if st is None:
            st = HostStreamer(self, chunks, slots)
            self.__dict__[key] = st
        outs = st.run(tuple(kinds), u, v, w, outs=out)
        torch.cuda.current_stream(self.device).synchronize()
        fl = int(st.flag.item())
        if fl & _lib.SEM1D_FLAG_STATE_NONFINITE:
            raise NumericFailure("state contains NaN/Inf")
        if fl & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
            raise NumericFailure("tangent contains NaN/Inf" if "jac" in kinds else "cotangent contains NaN/Inf")
        if host_np:
            return {k: t.numpy() for k, t in outs.items()}
        return outs

    def densify(self, u):
        """Dense J by columns (ops.py:259-273); verification only, n <= 5000."""
        torch = _torch()
        n = self.grid.nglobal
        if n > _DENSIFY_LIMIT:
            raise ValidationError(f"densify refused: {n} unknowns exceeds limit {_DENSIFY_LIMIT}")
        if self.batch != 1:
            raise ValidationError("densify needs batch == 1")
        ut, host = self.field(u, "state")
        cols = torch.empty((n, n), dtype=torch.float64, device=self.device)
        e = torch.zeros(n, dtype=torch.float64, device=self.device)
        col = self.empty()
        for k in range(n):
            e[k] = 1.0
            self.launch_jac(ut, e, col)
            cols[:, k] = col
            e[k] = 0.0
        self.counters["jac"] += n
        self.raise_for_flags(("state", "tangent"))
        return self._out(cols, host)


# -- streaming applies on host-resident fields -------------------------------------


class HostStreamer:
    """F / J v / J^T w on HOST fields, streamed through the GPU in element chunks.

    The ring is cut into C element blocks with the sharded ghost-element geometry of
    ``dist.Partition`` (each chunk recomputes its neighbours' boundary elements, so the
    result is bit-identical to the whole-ring apply).  Chunk i+1's host->device copies,
    chunk i's kernels and chunk i-1's device->host copies run on three streams, so a
    step costs max(H2D, D2H) instead of H2D + compute + D2H.  Inputs should be pinned
    CPU tensors (numpy arrays are staged through pinned buffers)."""

    def __init__(self, op, chunks=8, slots=3):
        import torch

        from .dist import Partition, shard_grid
        g = op.grid
        E = g.axis.elements
        chunks = max(2, min(int(chunks), E // 3))
        self.op, self.C = op, chunks
        self.parts = [Partition(E, g.axis.degree, chunks, c, g.periodic) for c in range(chunks)]
        self.ops = []
        cache = {}
        for p in self.parts:
            key = (p.E_ext, p.gl, p.gr, p.rank == 0, p.rank == chunks - 1)
            sg = shard_grid(g, p)
            # grids differ only in their extent; the plan depends on (E_ext, N, bc, h)
            k2 = (p.E_ext,)
            if k2 not in cache:
                cache[k2] = SemOperator(sg, op.coef, device=op.device, sync_checks=False)
            self.ops.append(cache[k2])
            del key
        self.flag = torch.zeros(1, dtype=torch.int32, device=op.device)
        for o in cache.values():
            o._flag = self.flag             # one flag word for the whole streamed apply
        self.maxext = max(p.ext_ndof for p in self.parts)
        self.ndof = g.nglobal
        dev = op.device
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        # device buffer sets: chunk c reuses set c % S once chunk c - S has left the
        # device, so S >= 3 keeps the H2D engine from waiting on the D2H of the
        # chunk just before it
        self.nslots = max(2, int(slots))
        self.slots = [{} for _ in range(self.nslots)]

    def _buf(self, slot, name):
        import torch
        b = self.slots[slot].get(name)
        if b is None:
            b = torch.empty(self.maxext, dtype=torch.float64, device=self.op.device)
            self.slots[slot][name] = b
        return b

    def _ranges(self, p):
        """(dst offset, src start, length) pieces of the chunk's ext range in the ring."""
        start = p.g_lo - p.gl * p.N
        n = p.ext_ndof
        out, off = [], 0
        while off < n:
            g = (start + off) % self.ndof
            ln = min(n - off, self.ndof - g)
            out.append((off, g, ln))
            off += ln
        return out

    def run(self, kinds, u, v=None, w=None, outs=None):
        """kinds: subset of ("rhs", "jac", "jact"); returns {kind: host tensor}."""
        import torch
        sync_copy = not u.is_pinned()   # pageable input: the copy engine cannot overlap it
        ins = {"u": u, "v": v, "w": w}
        outs = dict(outs or {})
        for k in kinds:
            if k not in outs:
                outs[k] = torch.empty(self.ndof, dtype=torch.float64, pin_memory=True)
        need = ["u"] + (["v"] if "jac" in kinds else []) + (["w"] if "jact" in kinds else [])
        uses = {"rhs": ("u",), "jac": ("u", "v"), "jact": ("u", "w")}
        ev_in = [{nm: torch.cuda.Event() for nm in need} for _ in range(self.C)]
        ev_out = [{k: torch.cuda.Event() for k in kinds} for _ in range(self.C)]
        ev_free = [torch.cuda.Event() for _ in range(self.C)]
        cur = torch.cuda.current_stream(self.op.device)
        self.s_h2d.wait_stream(cur)
        self.flag.zero_()
        S = self.nslots
        for c, p in enumerate(self.parts):
            slot = c % S
            op = self.ops[c]
            # per-field events: F(chunk c) starts, and its D2H leaves, as soon as u has
            # arrived, while v and w of the same chunk are still on the H2D engine
            with torch.cuda.stream(self.s_h2d):
                if c >= S:
                    self.s_h2d.wait_event(ev_free[c - S])      # slot's previous D2H done
                for name in need:
                    dst = self._buf(slot, name)
                    for off, g, ln in self._ranges(p):
                        dst[off:off + ln].copy_(ins[name][g:g + ln], non_blocking=not sync_copy)
                    ev_in[c][name].record(self.s_h2d)
            with torch.cuda.stream(self.s_cmp):
                n = p.ext_ndof
                ub = self._buf(slot, "u")[:n]
                for k in kinds:
                    self.s_cmp.wait_event(ev_in[c][uses[k][-1]])   # fields arrive in `need` order
                    ob = self._buf(slot, "o_" + k)[:n]
                    if k == "rhs":
                        op.launch_rhs(ub, ob)
                    elif k == "jac":
                        op.launch_jac(ub, self._buf(slot, "v")[:n], ob)
                    else:
                        op.launch_jact(ub, self._buf(slot, "w")[:n], ob)
                    ev_out[c][k].record(self.s_cmp)
            with torch.cuda.stream(self.s_d2h):
                sl = p.owned_slice()
                for k in kinds:
                    self.s_d2h.wait_event(ev_out[c][k])
                    outs[k][p.g_lo:p.g_lo + p.n_own].copy_(self._buf(slot, "o_" + k)[sl],
                                                           non_blocking=True)
                ev_free[c].record(self.s_d2h)
        cur.wait_stream(self.s_d2h)
        cur.wait_stream(self.s_cmp)
        self.op.counters.update({k: self.op.counters[k] + 1 for k in kinds})
        return outs


# -- grid maps on the device (used by Grid.scatter / Grid.gather) ----------------

_GEOM_PLANS = {}


def _geom_plan(grid, batch):
    key = (id(grid), batch)
    p = _GEOM_PLANS.get(key)
    if p is None:
        n = grid.axis.degree + 1
        z = np.zeros((n, n))
        p = _Plan(grid, 0.0, z, z, batch)
        _GEOM_PLANS[key] = (grid, p)   # keep grid alive while its plan is cached
        return p
    return p[1]


def _grid_scatter(grid, u):
    torch = _torch()
    host = not isinstance(u, torch.Tensor)
    t = torch.as_tensor(np.asarray(u, dtype=np.float64)) if host else u
    if tuple(t.shape) != (grid.nglobal,):
        raise ValidationError(f"field has shape {tuple(t.shape)}, expected ({grid.nglobal},)")
    if not t.is_cuda:
        t = t.cuda()
    t = t.contiguous().to(torch.float64)
    out = torch.empty((1, grid.nelem, grid.axis.degree + 1), dtype=torch.float64, device=t.device)
    p = _geom_plan(grid, 1)
    _lib.check(_lib.load().sem1d_scatter(p.handle, t.data_ptr(), out.data_ptr(),
                                         _stream_handle(t.device)), "sem1d_scatter")
    return out.cpu().numpy() if host else out


def _grid_gather(grid, local):
    torch = _torch()
    host = not isinstance(local, torch.Tensor)
    t = torch.as_tensor(np.asarray(local, dtype=np.float64)) if host else local
    want = (1, grid.nelem, grid.axis.degree + 1)
    if tuple(t.shape) != want:
        raise ValidationError(f"local block shape {tuple(t.shape)} does not match grid {want}")
    if not t.is_cuda:
        t = t.cuda()
    t = t.contiguous().to(torch.float64)
    out = torch.empty(grid.nglobal, dtype=torch.float64, device=t.device)
    p = _geom_plan(grid, 1)
    _lib.check(_lib.load().sem1d_gather(p.handle, t.data_ptr(), out.data_ptr(),
                                        _stream_handle(t.device)), "sem1d_gather")
    return out.cpu().numpy() if host else out
