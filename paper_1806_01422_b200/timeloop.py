"""Explicit-RK forward sweep on the B200 (reference ``semopt/timeloop.py``).

Every RK stage is ONE fused kernel (``sem1d_rk_stage``): it applies F to the
stage input and, in its epilogue, forms the next stage state (or the new
step state) from the base state and the stored slopes, so a step is s
launches and the stage temporaries of ``timeloop.py:111-130`` never exist.

Schemes: the reference's ``euler`` and ``rk3`` (Kutta-3, ``timeloop.py:24-27``)
with the reference's association order, plus ``rk4`` (classic tableau; absent
from the reference -- see DESIGN.md), and ``cn``: Crank-Nicolson by full Newton
with GMRES on (I - dt/2 J(v)) (``timeloop.py:133-186``), run natively by
``sem1d_cn_step`` (Newton + scipy-1.18.1 GMRES restated over the J kernel).
Adaptive Kutta-3 (``adaptive=True``) uses the embedded midpoint pair and the
controller of ``timeloop.py:198-218``; the weighted error is one device
reduction (``sem1d_rk_error_norm``), the accept / dt decision runs on the host.

Host control flow (dt clipping, StepFailure retries with dt halving,
snapshot selection) replicates ``timeloop.py:221-329`` exactly; the non-finite
checks of ``timeloop.py:100-103`` and ``ops.py:222-223`` come back as device
flag bits, read once per step.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import IntegrationError, NumericFailure, StepFailure, ValidationError

RK3_A = ((), (0.5,), (-1.0, 2.0))
RK3_B = (1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0)
RK3_BHAT = (0.0, 1.0, 0.0)
RK3_EMBEDDED_ORDER = 2

TABLEAUX = {
    "euler": (((),), (1.0,)),
    "rk3": (RK3_A, RK3_B),
    "rk4": (((), (0.5,), (0.0, 0.5), (0.0, 0.0, 1.0)), (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0)),
}

_RETRY_HALVINGS = 3   # timeloop.py:29
# fixed-dt runs on the fused step kernels verify their flags once per _SPEC_WINDOW steps;
# without stored snapshots the held states are capped at _SPEC_BYTES
_SPEC_WINDOW = 16
_SPEC_BYTES = 8e9


@dataclass
class TsConfig:
    """Time-stepper configuration (timeloop.py:32-76); ``rk4`` added."""

    scheme: str = "rk3"
    t0: float = 0.0
    t_end: float = 1.0
    dt: float = 0.01
    adaptive: bool = False
    tol_a: float = 1e-8
    tol_r: float = 1e-8
    alpha_min: float = 0.1
    alpha_max: float = 5.0
    beta: float = 0.9
    max_steps: int = 1_000_000
    newton_tol: float = 1e-10
    newton_max: int = 25
    gmres_tol: float = 1e-10
    gmres_max: int = 200
    gmres_restart: int = 30
    wlte_form: str = "rms"

    def __post_init__(self):
        self.validate()

    def validate(self):
        if self.scheme not in ("euler", "rk3", "rk4", "cn"):
            raise ValidationError(f"unknown scheme {self.scheme!r}")
        if not self.t_end > self.t0:
            raise ValidationError("t_end must exceed t0")
        if not self.dt > 0.0:
            raise ValidationError("dt must be positive")
        if not (0.0 < self.alpha_min < 1.0 < self.alpha_max):
            raise ValidationError("need 0 < alpha_min < 1 < alpha_max")
        if not (0.0 < self.beta < 1.0):
            raise ValidationError("need 0 < beta < 1")
        if self.adaptive and self.scheme != "rk3":
            raise ValidationError("adaptive stepping requires the embedded rk3 pair")
        if self.wlte_form not in ("rms", "max"):
            raise ValidationError(f"unknown wlte form {self.wlte_form!r}")


@dataclass
class ForwardResult:
    """Recorded trajectory (timeloop.py:79-97); states are device tensors."""

    ts: np.ndarray
    dts: np.ndarray
    snapshots: dict
    u_final: object
    stats: dict = field(default_factory=dict)
    step_log: list = field(default_factory=list)

    @property
    def n_steps(self):
        return len(self.dts)


def _require_explicit(cfg):
    """Batched / ring-resident sweeps run fixed-dt explicit schemes only."""
    if cfg.scheme == "cn":
        raise ValidationError("the batched ring-resident sweep runs explicit schemes only")
    if cfg.adaptive:
        raise ValidationError("the batched ring-resident sweep runs fixed-dt schemes only")


def _nonzero_terms(coefs, upto):
    return [(j, float(coefs[j])) for j in range(min(upto, len(coefs))) if coefs[j] != 0.0]


class StepEngine:
    """Launch plan + device scratch for one explicit step of a tableau.

    Stage kernel i computes k_i = F(U_i) and writes U_{i+1} (or, for the last
    stage, the new state) = base + dt * sum_j c_j k_j; slopes are stored only
    when a later combination reads them.
    """

    def __init__(self, op, scheme):
        if scheme not in TABLEAUX:
            raise ValidationError(f"unknown scheme {scheme!r}")
        self.op, self.scheme = op, scheme
        A, b = TABLEAUX[scheme]
        self.A, self.b, self.s = A, b, len(b)
        s = self.s
        # combination rows: row i+1 of A for stages, b for the step
        self.rows = [_nonzero_terms(A[i + 1], i + 1) for i in range(s - 1)]
        self.rows.append(_nonzero_terms(b, s))
        need = set()
        for i, row in enumerate(self.rows):
            for j, _ in row:
                if j < i:
                    need.add(j)
        self.stored_k = sorted(need)
        # stage recomputation (adjoint) only needs the A rows
        need_rec = set()
        for i, row in enumerate(self.rows[:-1]):
            for j, _ in row:
                if j < i:
                    need_rec.add(j)
        self.stored_k_recompute = sorted(need_rec)
        self._k = {}
        self._ping = None

    def _buf(self, key):
        t = self._k.get(key)
        if t is None:
            t = self.op.empty()
            self._k[key] = t
        return t

    def _launch_stage(self, i, U_in, base, dt, Y, check, store):
        row = self.rows[i]
        terms = [None if j == i else self._k[("k", j)] for j, _ in row]
        coefs = [c for _, c in row]
        k_out = self._buf(("k", i)) if i in store else None
        self.op.launch_rk_stage(U_in, k_out, base, terms, coefs, dt, Y, check)

    def step(self, u, dt, out, fused=True, stages_out=None, flag=None):
        """Launch one full step u -> out (no host sync): one temporally blocked launch
        when the ring qualifies (and ``fused``), else one fused launch per stage, which
        also leaves the stored slopes (k_2 of Kutta-3 for the embedded pair) in place.
        ``stages_out`` (fused path, s > 1): also write U_1..U_{s-1} there.  ``flag``
        (fused path): device address of the step's own flag word."""
        fz = getattr(self.op, "step_fused_supported", None)
        if fused and fz is not None and fz():
            kw = {} if flag is None else {"flag": flag}
            if stages_out is not None and self.s > 1:
                self.op.launch_rk_step_stages(u, out, stages_out, dt, self.scheme, **kw)
            else:
                self.op.launch_rk_step(u, out, dt, self.scheme, **kw)
            self.op.counters["rhs"] += self.s
            return
        s = self.s
        store = set(self.stored_k)
        for j in store:
            self._buf(("k", j))
        U = u
        for i in range(s):
            if i == s - 1:
                self._launch_stage(i, U, u, dt, out, True, store)
            else:
                Y = self._buf(("U", i % 2))
                self._launch_stage(i, U, u, dt, Y, False, store)
                U = Y
        self.op.counters["rhs"] += s

    def stages(self, u, dt, bufs):
        """Recompute stage states U_1..U_{s-1} into bufs[0..s-2]; returns [u, U_1, ...]."""
        s = self.s
        store = set(self.stored_k_recompute)
        for j in store:
            self._buf(("k", j))
        Us = [u]
        for i in range(s - 1):
            self._launch_stage(i, Us[-1], u, dt, bufs[i], False, store)
            Us.append(bufs[i])
        self.op.counters["rhs"] += s - 1
        return Us


def engine_for(op, scheme):
    cache = op.__dict__.setdefault("_engines", {})
    e = cache.get(scheme)
    if e is None:
        e = StepEngine(op, scheme)
        cache[scheme] = e
    return e


def check_step_flags(op):
    """Map device flags of one step to the reference exceptions."""
    v = op.flags()
    if v & (_lib.SEM1D_FLAG_STATE_NONFINITE | _lib.SEM1D_FLAG_INPUT2_NONFINITE):
        raise NumericFailure("state contains NaN/Inf")
    if v & _lib.SEM1D_FLAG_STEP_NONFINITE:
        raise StepFailure("state contains NaN/Inf")


def step_forward(op, u, t, dt, cfg, stats=None, out=None, check=True, fused=True):
    """One step of the configured scheme (timeloop.py:189-195); returns the new state."""
    if out is None:
        out = op.empty()
    if cfg.scheme == "cn":
        return step_cn(op, u, t, dt, cfg, stats, out=out)
    engine_for(op, cfg.scheme).step(u, dt, out, fused=fused)
    if check:
        check_step_flags(op)
    return out


def step_euler(op, u, t, dt):
    """One forward-Euler step (timeloop.py:106-108)."""
    ut, host = op.field(u, "state")
    out = op.empty()
    engine_for(op, "euler").step(ut, dt, out)
    check_step_flags(op)
    return out.cpu().numpy() if host else out


def step_rk3(op, u, t, dt):
    """One Kutta-3 step; returns (u_new, u_embedded, error_estimate) (timeloop.py:119-130).
    u_new comes from the per-stage kernels (k_2 stays on the device); the embedded
    midpoint u + dt k_2 and the difference are formed on the device."""
    ut, host = op.field(u, "state")
    e = engine_for(op, "rk3")
    u_new = op.empty()
    e.step(ut, dt, u_new, fused=False)
    check_step_flags(op)
    u_hat = ut + dt * e._k[("k", 1)]
    err = u_new - u_hat
    if host:
        return u_new.cpu().numpy(), u_hat.cpu().numpy(), err.cpu().numpy()
    return u_new, u_hat, err


def _cn_raise(st, what):
    """Map sem1d_cn_stats.status to the reference exceptions (timeloop.py:146-186)."""
    s = st.status
    if s == _lib.SEM1D_CN_OK:
        return
    if s == _lib.SEM1D_CN_GMRES_FAILED:
        raise StepFailure(f"GMRES did not converge (info={st.gmres_info})",
                          diagnostics={"gmres_info": st.gmres_info, "gmres_iters": st.gmres_iters})
    if s == _lib.SEM1D_CN_NEWTON_STALLED:
        raise StepFailure(f"Newton stalled after {st.newton_iters} iterations "
                          f"(|r|={st.last_residual:.3e})", diagnostics={"newton_iters": st.newton_iters})
    if s == _lib.SEM1D_CN_RESIDUAL_NONFINITE:
        raise StepFailure("residual contains NaN/Inf")
    raise NumericFailure(f"{what} contains NaN/Inf")


def step_cn(op, u, t, dt, cfg, stats=None, out=None):
    """One Crank-Nicolson step (timeloop.py:154-186) on the device: full Newton with the
    Jacobian re-evaluated each iteration, unpreconditioned GMRES on (I - dt/2 J(v)).
    ``stats`` receives newton_iters (successful steps only) and gmres_iters, as in the
    reference; StepFailure / NumericFailure as the reference raises them."""
    if not hasattr(op, "launch_cn_step"):
        raise ValidationError("Crank-Nicolson runs on a single-device batch-1 SemOperator")
    ut, host = op.field(u, "state")
    out = op.empty() if out is None else out
    st = _lib.CnStats()
    op.launch_cn_step(ut, out, dt, cfg, st)
    op.counters["rhs"] += st.rhs_applies
    op.counters["jac"] += st.jac_applies
    if stats is not None:
        stats["gmres_iters"] = stats.get("gmres_iters", 0) + st.gmres_iters
    _cn_raise(st, "state")
    if stats is not None:
        stats["newton_iters"] = stats.get("newton_iters", 0) + st.newton_iters
    return out.cpu().numpy() if host else out


def controller(err, u_new, u_hat, dt_old, cfg):
    """Embedded-pair step-size controller (timeloop.py:198-218) on numpy arrays or
    device tensors; ``integrate`` uses the fused device reduction instead."""
    xp = np
    if not isinstance(err, np.ndarray):
        import torch as xp  # noqa: N812
    tol = cfg.tol_a + xp.maximum(xp.abs(u_new), xp.abs(u_hat)) * cfg.tol_r
    ratios = xp.abs(err) / tol
    wlte = float(xp.mean(xp.sqrt(ratios))) if cfg.wlte_form == "rms" else float(xp.max(ratios))
    return _controller_decision(wlte, dt_old, cfg)


def _controller_decision(wlte, dt_old, cfg):
    if wlte == 0.0:
        return True, cfg.alpha_max * dt_old, wlte
    factor = min(cfg.alpha_max,
                 max(cfg.alpha_min, cfg.beta * (1.0 / wlte) ** (1.0 / (RK3_EMBEDDED_ORDER + 1))))
    return wlte <= 1.0, factor * dt_old, wlte


def count_steps(cfg):
    """Number of fixed-dt steps (timeloop.py:221-234)."""
    if cfg.adaptive:
        raise ValidationError("step count of an adaptive run is not known a priori")
    tiny = 1e-9 * cfg.dt
    t, n = cfg.t0, 0
    while t < cfg.t_end - tiny:
        clipped = (cfg.t_end - t) - cfg.dt <= tiny
        t = cfg.t_end if clipped else t + cfg.dt
        n += 1
        if n > cfg.max_steps:
            raise ValidationError(f"fixed-dt run exceeds max_steps={cfg.max_steps}")
    return n


def stages_supported(op, cfg):
    """Whether a forward run can hold its stage states in HBM for the adjoint (fused
    whole-step kernels, explicit multi-stage scheme, fixed dt)."""
    fz = getattr(op, "step_stages_supported", None)
    return (cfg.scheme in TABLEAUX and len(TABLEAUX[cfg.scheme][1]) > 1 and not cfg.adaptive
            and fz is not None and fz())


def integrate(op, u0, cfg, store_steps="all", keep_log=False, keep_stages=False):
    """Integrate t0 -> t_end recording the trajectory (timeloop.py:237-329).

    ``store_steps``: "all", an iterable of step indices, or None (step 0 only).
    Stored states stay on the device; a StepFailure is retried with dt halved
    up to three times, exactly like the reference.
    """
    u, _ = op.field(u0, "initial state")
    if not bool(op._isfinite_all(u)):
        raise NumericFailure("initial state contains NaN/Inf")
    store_all = store_steps == "all"
    want = None if store_all else ({0} if store_steps is None else {int(s) for s in store_steps})
    stats = {"steps": 0, "rejects": 0, "retries": 0, "newton_iters": 0, "gmres_iters": 0}
    snapshots = {}
    if store_all or 0 in want:
        snapshots[0] = u.clone()
    ts, dts = [cfg.t0], []
    log = [] if keep_log else None
    t, dt_next = cfg.t0, cfg.dt
    tiny = 1e-9 * cfg.dt
    n = attempts = 0
    cn = cfg.scheme == "cn"
    engine = None if cn else engine_for(op, cfg.scheme)
    fused = not cfg.adaptive          # the embedded pair needs the per-stage k_2
    # stage states held in HBM for the adjoint (north_star item 4): a step that starts from
    # a stored state keeps U_1..U_{s-1}; the sweep then skips the stage recompute
    keep_stages = bool(keep_stages) and stages_supported(op, cfg)
    stage_snaps = {}
    op.flags()  # clear stale bits
    # Running ahead (fixed-dt explicit schemes on the fused step kernels): up to `window` steps
    # are launched without a host sync, each OR-ing its non-finite bits into its own flag
    # word; the window is then verified with ONE device->host read.  A flagged step j rolls
    # the run back to the state before j (trajectory, counters and log included) and step j is
    # re-run synchronously, so StepFailure retries / NumericFailure behave exactly as in the
    # per-step-checked loop.  Without stored snapshots the window's states are held for the
    # rollback, so the window is sized to the free-memory budget.
    fz = getattr(op, "step_fused_supported", None)
    spec = (not cn and fused and getattr(op, "supports_flag_slots", False) and fz is not None and fz())
    window = 0
    if spec:
        field_bytes = 8 * int(op.empty().numel())
        window = _SPEC_WINDOW if store_all else max(0, min(_SPEC_WINDOW, int(_SPEC_BYTES // field_bytes)))
        spec = window >= 2
    if spec:
        slots = op.flag_slots(window)
        slots.zero_()
        slot0 = slots.data_ptr()
    pending = []            # rollback records of the launched, unverified steps
    sync_next = False       # re-run the next step with a per-step check (after a rollback)

    def verify():
        """Check the pending window; on a flagged step roll back to it.  True if rolled back."""
        nonlocal n, t, dt_next, attempts, u, sync_next
        words = slots[:len(pending)]
        red = getattr(op, "reduce_flag_words", None)      # sharded: agree across ranks
        vals = (red(words) if red is not None else words).cpu().tolist()
        slots.zero_()
        bad = next((i for i, v in enumerate(vals) if v), None)
        if bad is None:
            pending.clear()
            return False
        n, t, dt_next, attempts, u, nlog, counters = pending[bad]
        op.counters.clear()
        op.counters.update(counters)          # the discarded steps were never taken
        for rec in pending[bad:]:
            snapshots.pop(rec[0] + 1, None)
            stage_snaps.pop(rec[0], None)
        del ts[n + 1:]
        del dts[n:]
        if keep_log:
            del log[nlog:]
        stats["steps"] = n
        pending.clear()
        sync_next = True
        return True

    while t < cfg.t_end - tiny:
        attempts += 1
        if attempts > cfg.max_steps:
            if spec and pending and verify():
                continue
            raise IntegrationError(f"max_steps={cfg.max_steps} exceeded at t={t:.6g}",
                                   diagnostics={"t": t, "steps": n, "stats": stats})
        remaining = cfg.t_end - t
        clipped = remaining - dt_next <= tiny
        dt = remaining if clipped else dt_next
        u_new = op.empty()
        if spec and not sync_next:
            keep_n = keep_stages and (store_all or n in want)
            st_out = [op.empty() for _ in range(engine.s - 1)] if keep_n else None
            pending.append((n, t, dt_next, attempts - 1, u, len(log) if keep_log else 0, dict(op.counters)))
            engine.step(u, dt, u_new, fused=True, stages_out=st_out, flag=slot0 + 4 * (len(pending) - 1))
            if keep_n:
                stage_snaps[n] = st_out
            n += 1
            t = cfg.t_end if clipped else t + dt
            dts.append(dt)
            ts.append(t)
            u = u_new
            stats["steps"] = n
            if store_all or n in want:
                snapshots[n] = u
            if keep_log:
                log.append((n, t, dt, 0.0, 1))
            if len(pending) == window or not t < cfg.t_end - tiny:
                verify()
            continue
        sync_next = False
        for retry in range(_RETRY_HALVINGS + 1):
            try:
                if cn:
                    step_cn(op, u, t, dt, cfg, stats, out=u_new)
                else:
                    keep_n = keep_stages and (store_all or n in want)   # the step from a kept state
                    st_out = [op.empty() for _ in range(engine.s - 1)] if keep_n else None
                    engine.step(u, dt, u_new, fused=fused, stages_out=st_out)
                    check_step_flags(op)
                    if keep_n:
                        stage_snaps[n] = st_out
                break
            except StepFailure:
                stats["retries"] += 1
                if retry == _RETRY_HALVINGS:
                    raise
                dt *= 0.5
                clipped = False
        wlte = 0.0
        if cfg.adaptive:
            wlte = op.rk_error_norm(u_new, u, engine._k[("k", 1)], dt, cfg)
            accept, dt_prop, wlte = _controller_decision(wlte, dt, cfg)
            if not accept:
                stats["rejects"] += 1
                if keep_log:
                    log.append((n, t, dt, wlte, 0))
                dt_next = dt_prop
                continue
            dt_next = dt_prop
        elif dt != dt_next and not clipped:
            dt_next = dt
        n += 1
        t = cfg.t_end if clipped else t + dt
        dts.append(dt)
        ts.append(t)
        u = u_new
        stats["steps"] = n
        if store_all or n in want:
            snapshots[n] = u
        if keep_log:
            log.append((n, t, dt, wlte, 1))
    res = ForwardResult(ts=np.asarray(ts), dts=np.asarray(dts), snapshots=snapshots,
                        u_final=u, stats=stats, step_log=log if keep_log else [])
    res.fused_steps = fused       # replays (checkpoint Advance) take the same kernel path
    res.stage_snapshots = stage_snaps
    return res


def rk3_stages(op, u, t, dt):
    """Stage states (U1, U2, U3) of the Kutta-3 step (timeloop.py:111-117)."""
    e = engine_for(op, "rk3")
    bufs = [op.empty(), op.empty()]
    Us = e.stages(u, dt, bufs)
    check_step_flags(op)
    return tuple(Us)


def fixed_step_sizes(cfg):
    """The dt sequence of a fixed-dt run (timeloop.py:264-278, no failures)."""
    tiny = 1e-9 * cfg.dt
    t, dts = cfg.t0, []
    while t < cfg.t_end - tiny:
        remaining = cfg.t_end - t
        clipped = remaining - cfg.dt <= tiny
        dt = remaining if clipped else cfg.dt
        t = cfg.t_end if clipped else t + dt
        dts.append(dt)
        if len(dts) > cfg.max_steps:
            raise ValidationError(f"fixed-dt run exceeds max_steps={cfg.max_steps}")
    return dts


def ring_resident_supported(op):
    """Whether the whole ring fits one CTA (mirrors launch_ens_forward in csrc)."""
    if getattr(op.coef, "advection", "burgers") != "burgers" or op.grid.dim != 1:
        return False                     # the ring-resident kernels implement 1D Burgers
    ax = op.grid.axis
    E, n = ax.elements, ax.degree + 1
    if E * n <= 1024:
        return True
    return bool(op.grid.periodic and n % 8 == 0 and E % 8 == 0 and E <= 256)


def _dts_device(op, cfg):
    """The fixed-dt sequence on the host and on the device, cached per operator and
    time grid (the ring-resident sweeps of small problems are latency-bound)."""
    import torch
    key = (cfg.t0, cfg.t_end, cfg.dt, cfg.max_steps)
    cache = op.__dict__.setdefault("_dts_cache", {})
    hit = cache.get(key)
    if hit is None:
        dts = fixed_step_sizes(cfg)
        hit = (dts, torch.tensor(dts, dtype=torch.float64, device=op.device))
        if len(cache) > 16:
            cache.clear()
        cache[key] = hit
    return hit


def integrate_ensemble(op, u0, cfg, store_trajectory=True, defer_checks=False):
    """Forward sweep of a batch of independent rings, one CTA per ring, every step in
    shared memory (sem1d_ens_forward).  Same dt sequence and step arithmetic as
    :func:`integrate`; a problem whose state goes non-finite is reported in
    ``stats["failed"]`` (the batched sweep does not retry with halved dt).
    ``defer_checks``: no host sync here -- the result carries ``flags_device`` and
    ``initial_ok_device`` and ``stats["failed"]`` is None until the caller reads them
    (``AssimilationProblem.evaluate`` reads every check of a gradient in one transfer)."""
    import torch
    _require_explicit(cfg)
    u, _ = op.field(u0, "initial state")
    init_ok = None
    if defer_checks:
        init_ok = torch.isfinite(u).all()
    elif not op._isfinite_all(u):
        raise NumericFailure("initial state contains NaN/Inf")
    dts, dts_dev = _dts_device(op, cfg)
    m = len(dts)
    traj = None
    if store_trajectory:
        traj = torch.empty((m + 1,) + tuple(u.shape), dtype=torch.float64, device=op.device)
    u_final = op.empty()
    flags = torch.zeros(op.batch, dtype=torch.int32, device=op.device)
    op.launch_ens_forward(u.contiguous(), traj, u_final, dts_dev, m, cfg.scheme, flags)
    op.counters["rhs"] += len(TABLEAUX[cfg.scheme][1]) * m
    failed = None
    if not defer_checks:
        fl = flags.cpu()
        failed = [int(i) for i in torch.nonzero(fl).flatten()]
    snapshots = {n: traj[n] for n in range(m + 1)} if traj is not None else {0: u.clone()}
    ts = np.concatenate([[cfg.t0], cfg.t0 + np.cumsum(dts)]) if m else np.asarray([cfg.t0])
    if m:
        ts[-1] = cfg.t_end
    stats = {"steps": m, "rejects": 0, "retries": 0, "failed": failed}
    res = ForwardResult(ts=ts, dts=np.asarray(dts), snapshots=snapshots, u_final=u_final,
                        stats=stats)
    res.trajectory = traj          # (m+1, batch, ndof) step-major, for ensemble_sweep
    res.dts_device = dts_dev
    res.flags_device = flags
    res.initial_ok_device = init_ok
    return res
