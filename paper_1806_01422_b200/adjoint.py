"""Discrete-adjoint backward sweep on the B200 (reference ``semopt/adjoint.py``).

Crank-Nicolson steps transpose through ``sem1d_cn_adjoint_step``: GMRES with J^T
applications only, (I - dt/2 J(u_{n+1}))^T mu = lam, then lam_n = mu + dt/2 J^T(u_n) mu
(adjoint.py:64-69).

One adjoint step of an s-stage explicit scheme is 2s-1 fused launches: s-1
``sem1d_rk_stage`` kernels recompute the stage states from the checkpointed
u_n (adjoint.py:56), then s ``sem1d_adj_stage`` kernels run the stage-adjoint
recurrence of adjoint.py:58-61, generalised to any tableau,

    l_i = dt J^T(U_i) (b_i lam + sum_{j>i} a_ji l_j),   lam' = lam + l_1 + ... + l_s,

each forming its J^T input while staging the slab and folding dt and the
final accumulation into its epilogue.  ``sweep`` interprets the reference
checkpoint schedules (checkpoint.py) over device-resident slots.
"""

from __future__ import annotations

from . import _lib
from .checkpoint import Advance, AdjointStep, Done, Restore, Store
from .errors import CheckpointError, NumericFailure, ValidationError
from .timeloop import TABLEAUX, _cn_raise, check_step_flags, engine_for, step_cn


def terminal_condition(grid, u_final, u_ref, op=None):
    """(J, lam_N) with J = d^T M d, lam_N = mask(2 M d), d = u_final - u_ref (adjoint.py:33-47).

    Runs as one fused reduction kernel pair on the device (needs ``op`` or an
    operator cached on the grid)."""
    import torch
    op = op or getattr(grid, "_default_op", None)
    if op is None:
        raise ValidationError("terminal_condition on the B200 path needs the operator (op=...)")
    uN, host = op.field(u_final, "misfit")
    ud, _ = op.field(u_ref, "misfit")
    lam = op.empty()
    J = torch.empty(op.batch, dtype=torch.float64, device=op.device)
    op.launch_terminal(uN, ud, lam, J)
    if op.batch == 1:
        j = float(J.item())
        return j, (lam.cpu().numpy() if host else lam)
    return J, lam


class AdjointEngine:
    """Device scratch + launch plan for one backward step of a tableau."""

    def __init__(self, op, scheme):
        self.op, self.scheme = op, scheme
        A, b = TABLEAUX[scheme]
        self.A, self.b, self.s = A, b, len(b)
        self.fwd = engine_for(op, scheme)
        self._U = None
        self._L = None
        # z-combination terms of stage i: (a_ji, j) for j > i with a_ji != 0
        self.zterms = []
        for i in range(self.s):
            terms = []
            for j in range(i + 1, self.s):
                a = A[j][i] if i < len(A[j]) else 0.0
                if a != 0.0:
                    terms.append((j, float(a)))
            self.zterms.append(terms)

    @property
    def U(self):   # per-stage scratch, allocated only if the per-stage path runs
        if self._U is None:
            self._U = [self.op.empty() for _ in range(self.s - 1)]
        return self._U

    @property
    def L(self):
        if self._L is None:
            self._L = {i: self.op.empty() for i in range(1, self.s)}
        return self._L

    def step(self, u_n, lam, dt, lam_out, stages=None, flag=None):
        """lam_out = transpose of the step map at u_n applied to lam (no host sync).
        ``stages``: the step's stage states U_1..U_{s-1} stored by the forward run (fused
        path): no recompute.  ``flag``: device address of this step's own flag word (fused
        path, ``sweep`` running ahead); default the operator's flag."""
        op, s = self.op, self.s
        fused = getattr(op, "step_fused_supported", None)
        if fused is not None and fused():
            kw = {} if flag is None else {"flag": flag}
            if stages is not None and s > 1:
                op.launch_adj_step_stages(u_n, stages, lam, lam_out, dt, self.scheme, **kw)
            else:
                op.launch_adj_step(u_n, lam, lam_out, dt, self.scheme, **kw)
                op.counters["rhs"] += s - 1
            op.counters["jact"] += s
            return
        Us = self.fwd.stages(u_n, dt, self.U) if s > 1 else [u_n]
        for i in range(s - 1, -1, -1):
            lts = [self.L[j] for j, _ in self.zterms[i]]
            acs = [a for _, a in self.zterms[i]]
            if i > 0:
                op.launch_adj_stage(Us[i], lam, self.b[i], lts, acs, dt, self.L[i], None, None)
            else:
                acc = [None] + [self.L[j] for j in range(1, s)]
                op.launch_adj_stage(Us[0], lam, self.b[0], lts, acs, dt, None, acc, lam_out)
        op.counters["jact"] += s


def resolve_ensemble_flags(op, cfg, fwd, lam_terminal, word):
    """An outputs-only ensemble sweep flagged a problem: classify it with a re-run of the
    sweep under the per-stage cotangent checks (counters untouched) and raise the reference's
    NumericFailure if a cotangent was non-finite; a flag from an overflow of the final
    gradient alone returns (the reference raises only when a later apply reads it)."""
    import torch
    word = int(word)
    if not word & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
        saved = dict(op.counters)
        lam_in, _ = op.field(lam_terminal, "cotangent")
        flags = torch.zeros(op.batch, dtype=torch.int32, device=op.device)
        op.launch_ens_adjoint(fwd.trajectory, lam_in.contiguous(), op.empty(), fwd.dts_device, fwd.n_steps,
                              cfg.scheme, flags, check=True)
        word = int(flags.max())
        op.counters.clear()
        op.counters.update(saved)
    if word & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
        raise NumericFailure("cotangent contains NaN/Inf")


def adjoint_engine_for(op, scheme):
    cache = op.__dict__.setdefault("_adj_engines", {})
    e = cache.get(scheme)
    if e is None:
        e = AdjointEngine(op, scheme)
        cache[scheme] = e
    return e


def _check_adjoint_flags(op, v=None):
    v = op.flags() if v is None else v
    if v & _lib.SEM1D_FLAG_STATE_NONFINITE:
        raise NumericFailure("state contains NaN/Inf")
    if v & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
        raise NumericFailure("cotangent contains NaN/Inf")


def adjoint_step(op, u_n, lam, t, dt, scheme, out=None):
    out = op.empty() if out is None else out
    adjoint_engine_for(op, scheme).step(u_n, lam, dt, out)
    _check_adjoint_flags(op)
    return out


def adjoint_step_cn(op, u_n, u_np1, lam, t, dt, cfg, stats=None, out=None):
    """Transpose of one CN step (adjoint.py:64-69) on the device; ``stats`` receives
    gmres_iters; GMRES non-convergence raises StepFailure like the reference."""
    from . import _lib
    if not hasattr(op, "launch_cn_adjoint_step"):
        raise ValidationError("Crank-Nicolson runs on a single-device batch-1 SemOperator")
    un, host = op.field(u_n, "state")
    up, _ = op.field(u_np1, "state")
    lt, _ = op.field(lam, "cotangent")
    out = op.empty() if out is None else out
    st = _lib.CnStats()
    op.launch_cn_adjoint_step(un, up, lt, out, dt, cfg, st)
    op.counters["jact"] += st.jact_applies
    if stats is not None:
        stats["gmres_iters"] = stats.get("gmres_iters", 0) + st.gmres_iters
    _cn_raise(st, "cotangent")
    return out.cpu().numpy() if host else out


_ADJ_WINDOW = 16      # adjoint steps launched between two flag reads (run-ahead sweep)
_ADJ_WINDOW_BYTES = 8e9   # cotangents a run-ahead window keeps alive for a classifying re-run


def sweep(op, cfg, fwd, schedule, lam_terminal, check_every=None):
    """Backward sweep over a recorded trajectory (adjoint.py:72-158).

    Schedule semantics, CheckpointError conditions and ``last_sweep_stats``
    follow the reference; states are device tensors, a Store keeps a
    reference (states are never mutated in place), an Advance re-runs the
    recorded dts through the same fused stage kernels (bitwise replay).

    Flags: on the fused step kernels the sweep runs ahead (``check_every=None``): each
    adjoint step tests only its output cotangent and ORs the result into its own flag word,
    and one device->host read verifies up to _ADJ_WINDOW steps (and always before a
    recompute Advance and at the end).  A flagged step is re-run from its kept inputs with
    the classifying check (state / cotangent, as the reference's per-call checks), bitwise
    the same output; the first step that classifies raises the same NumericFailure, with the
    same counters, as the per-step check (``check_every=1``) would have.
    """
    m = fwd.n_steps
    if schedule.n_steps != m:
        raise ValidationError(f"schedule covers {schedule.n_steps} steps, trajectory has {m}")
    lam_t, host = op.field(lam_terminal, "cotangent")
    lam = lam_t.clone()
    if m == 0:
        return lam.cpu().numpy() if host else lam
    dts = fwd.dts
    stats = {"newton_iters": 0, "gmres_iters": 0, "recomputed": 0}
    cn = cfg.scheme == "cn"
    fwd_engine = None if cn else engine_for(op, cfg.scheme)
    adj = None if cn else adjoint_engine_for(op, cfg.scheme)
    fused = getattr(fwd, "fused_steps", True)   # replay with the forward run's kernel path
    stage_snaps = getattr(fwd, "stage_snapshots", None) or {}   # stage states kept in HBM

    slots, preloaded = {}, True
    for step, slot in schedule.forward_stores.items():
        if step in fwd.snapshots:
            slots[slot] = (step, fwd.snapshots[step])
        else:
            preloaded = False
    if preloaded:
        actions = schedule.actions[schedule.backward_start:]
        current = None
    else:
        if 0 not in fwd.snapshots:
            raise CheckpointError("trajectory does not retain the initial state")
        slots = {}
        actions = schedule.actions
        current = (0, fwd.snapshots[0])

    succ = (m, fwd.u_final)
    next_adj = m - 1
    spare = op.empty()
    since_check = 0
    op.flags()
    fz = getattr(op, "step_fused_supported", None)
    ahead = (check_every is None and not cn and getattr(op, "supports_flag_slots", False)
             and fz is not None and fz())
    check_every = 1 if check_every is None else check_every
    # unverified steps: (step, counters after it, u_n, lam_{n+1}, stages, dt) -- the inputs
    # stay alive until the window is verified, for the classifying re-run of a flagged step
    pending = []
    window = _ADJ_WINDOW
    if ahead:
        field = max(1, op.ndof * getattr(op, "batch", 1) * 8)
        window = max(1, min(_ADJ_WINDOW, int(_ADJ_WINDOW_BYTES // field)))
        wslots = op.flag_slots(window)
        wslots.zero_()
        wslot0 = wslots.data_ptr()
    classify = _lib.SEM1D_FLAG_STATE_NONFINITE | _lib.SEM1D_FLAG_INPUT2_NONFINITE

    def verify():
        if not pending:
            return
        words = wslots[:len(pending)]
        red = getattr(op, "reduce_flag_words", None)      # sharded: OR over ranks
        vals = (red(words) if red is not None else words).cpu().tolist()
        wslots.zero_()
        for j, v in enumerate(vals):
            if not v:
                continue
            n, after, u_j, lam_j, st_j, dt_j = pending[j]
            if not v & classify:
                # outputs-only flag: re-run the step with the classifying check (the op's own
                # flag word; sharded ranks all take this branch: the words were OR-reduced)
                saved = dict(op.counters)
                op.flags()
                adj.step(u_j, lam_j, dt_j, op.empty(), stages=st_j)
                v = op.flags()
                op.counters.clear()
                op.counters.update(saved)
            if v & classify:
                op.counters.clear()
                op.counters.update(after)                # as if the sweep stopped at that step
                pending.clear()
                _check_adjoint_flags(op, v)
            # an output that overflowed from finite inputs: the reference raises only when a
            # later step reads it as its cotangent, which that step's re-run classifies
        pending.clear()

    for act in actions:
        if isinstance(act, Restore):
            if act.slot not in slots or slots[act.slot][0] != act.step:
                raise CheckpointError(f"restore of step {act.step}: slot not populated")
            current = slots[act.slot]
        elif isinstance(act, Store):
            if current is None or current[0] != act.step:
                raise CheckpointError(f"store at step {act.step}: state not in hand")
            slots[act.slot] = current
        elif isinstance(act, Advance):
            if current is None or current[0] != act.start:
                raise CheckpointError(f"advance from step {act.start}: state not in hand")
            if ahead:
                verify()                   # the per-step loop would have raised before this
            u = current[1]
            for n in range(act.start, act.stop):
                nxt = op.empty()
                if cn:
                    step_cn(op, u, fwd.ts[n], dts[n], cfg, stats, out=nxt)
                else:
                    fwd_engine.step(u, dts[n], nxt, fused=fused)
                u = nxt
            if not cn:
                check_step_flags(op)
            stats["recomputed"] += act.stop - act.start
            current = (act.stop, u)
        elif isinstance(act, AdjointStep):
            n = act.step
            if n != next_adj:
                raise CheckpointError(f"adjoint step {n} out of order")
            if current is None or current[0] != n:
                raise CheckpointError(f"adjoint step {n}: forward state missing")
            if not (succ[0] == n + 1 or n + 1 == m):
                raise CheckpointError(f"adjoint step {n}: successor state missing")
            if cn:
                u_np1 = succ[1] if succ[0] == n + 1 else fwd.u_final
                adjoint_step_cn(op, current[1], u_np1, lam, fwd.ts[n], dts[n], cfg, stats, out=spare)
            elif ahead:
                spare = op.empty()                       # lam stays alive while the step is pending
                adj.step(current[1], lam, dts[n], spare, stages=stage_snaps.get(n),
                         flag=wslot0 + 4 * len(pending))
                pending.append((n, dict(op.counters), current[1], lam, stage_snaps.get(n), dts[n]))
            else:
                adj.step(current[1], lam, dts[n], spare, stages=stage_snaps.get(n))
            lam, spare = spare, lam
            if ahead:
                if len(pending) == window:
                    verify()
            else:
                since_check += 1
                if since_check >= check_every:
                    _check_adjoint_flags(op)
                    since_check = 0
            succ = current
            next_adj -= 1
        elif isinstance(act, Done):
            break
    if ahead:
        verify()
    _check_adjoint_flags(op)
    if next_adj != -1:
        raise CheckpointError(f"sweep incomplete: stopped before adjoint step {next_adj}")
    op.last_sweep_stats = stats
    return lam.cpu().numpy() if host else lam


def gradient(op, cfg, fwd, schedule, u_ref):
    """terminal_condition + sweep (adjoint.py:161-164)."""
    j, lam = terminal_condition(op.grid, fwd.u_final, u_ref, op=op)
    return j, sweep(op, cfg, fwd, schedule, lam)


def ensemble_sweep(op, cfg, fwd, lam_terminal, defer_checks=False, check=False):
    """Backward sweep of a batch of rings over a trajectory from
    ``timeloop.integrate_ensemble`` -- one CTA per ring, every step in shared memory
    (sem1d_ens_adjoint).  Same recurrence as :func:`sweep` with store-all; the stage
    adjoints are accumulated as lam + (l_s + ... + l_1) instead of ((lam + l_1) + ...).
    The sweep tests only its outputs; a flagged sweep is re-run with the classifying check
    (``check=True``, every stage's cotangent) and raises NumericFailure("cotangent ...") only
    if a cotangent was non-finite -- a final overflow alone is returned, as the reference's
    sweep would.  ``defer_checks``: returns (gradient, per-problem flag words on the device)
    without a host sync; the caller resolves them (:func:`resolve_ensemble_flags`)."""
    import torch
    traj = getattr(fwd, "trajectory", None)
    if traj is None:
        raise ValidationError("ensemble_sweep needs the stored trajectory of integrate_ensemble")
    lam_in, host = op.field(lam_terminal, "cotangent")
    lam_out = op.empty()
    flags = torch.zeros(op.batch, dtype=torch.int32, device=op.device)
    op.launch_ens_adjoint(traj, lam_in.contiguous(), lam_out, fwd.dts_device, fwd.n_steps,
                          cfg.scheme, flags, check=check)
    if not defer_checks and int(flags.max()):
        resolve_ensemble_flags(op, cfg, fwd, lam_in, flags.max())
    s = len(TABLEAUX[cfg.scheme][1])
    op.counters["rhs"] += (s - 1) * fwd.n_steps
    op.counters["jact"] += s * fwd.n_steps
    op.last_sweep_stats = {"newton_iters": 0, "gmres_iters": 0, "recomputed": 0}
    if defer_checks:
        return lam_out, flags
    return lam_out.cpu().numpy() if host else lam_out
