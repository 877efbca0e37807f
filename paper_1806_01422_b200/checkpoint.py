"""Trajectory checkpoint schedules (reference ``semopt/checkpoint.py``).

Host-only planning; the sweep (adjoint.py) executes the actions over device
slots.  Schedules are identical, action for action, to the reference's
(checked against ``tests/golden/schedules.npz``): same DP recurrence for the
optimal recomputation count (checkpoint.py:93-135) and the same tie rule
(smallest first-checkpoint offset that strictly beats the no-checkpoint
cost).  The DP is evaluated bottom-up with vectorised minima and the
emission is iterative, so long horizons (m = 500, s = 64 for BASELINE
config 5) plan in well under a second and never hit Python's recursion limit.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .errors import ScheduleError, ValidationError


@dataclass(frozen=True)
class Store:
    slot: int
    step: int


@dataclass(frozen=True)
class Restore:
    slot: int
    step: int


@dataclass(frozen=True)
class Advance:
    start: int
    stop: int


@dataclass(frozen=True)
class AdjointStep:
    step: int


@dataclass(frozen=True)
class Done:
    pass


@dataclass
class Schedule:
    n_steps: int
    slots: int
    actions: list
    recomputed: int
    forward_stores: dict = field(default_factory=dict)  # step -> slot
    backward_start: int = 0


def plan_store_all(m):
    """Keep every state 0..m-1 (checkpoint.py:70-90)."""
    if m < 1:
        raise ValidationError("need at least one step")
    acts = []
    for n in range(m):
        acts += [Store(n, n), Advance(n, n + 1)]
    start = len(acts)
    for n in range(m - 1, -1, -1):
        acts += [Restore(n, n), AdjointStep(n)]
    acts.append(Done())
    return Schedule(n_steps=m, slots=m, actions=acts, recomputed=0,
                    forward_stores={n: n for n in range(m)}, backward_start=start)


@lru_cache(maxsize=64)
def _tables(m, f_max):
    """Bottom-up DP over chain length l <= m and free slots f <= f_max.

    back[l, f]:  advances to adjoint a chain of l steps, left state held, f free slots;
    total[l, f]: same, but the chain end must be reached once first;
    kb / kt:     the optimal first-checkpoint offset (-1 = none)."""
    back = np.zeros((m + 1, f_max + 1), dtype=np.int64)
    total = np.zeros((m + 1, f_max + 1), dtype=np.int64)
    kb = np.full((m + 1, f_max + 1), -1, dtype=np.int64)
    kt = np.full((m + 1, f_max + 1), -1, dtype=np.int64)
    if m >= 1:
        total[1, :] = 1
    for f in range(f_max + 1):
        for l in range(2, m + 1):
            base_b = l * (l - 1) // 2
            base_t = l + back[l, f]   # back[l, f] is final before total[l, f] is needed
            if f >= 1:
                ks = np.arange(1, l)
                cb = ks + back[l - ks, f - 1] + back[ks, f]
                i = int(np.argmin(cb))
                if cb[i] < base_b:
                    back[l, f], kb[l, f] = cb[i], i + 1
                else:
                    back[l, f] = base_b
                base_t = l + back[l, f]
                ct = ks + total[l - ks, f - 1] + back[ks, f]
                i = int(np.argmin(ct))
                if ct[i] < base_t:
                    total[l, f], kt[l, f] = ct[i], i + 1
                else:
                    total[l, f] = base_t
            else:
                back[l, f] = base_b
                total[l, f] = l + base_b
    return back, total, kb, kt


def binomial_cost(m, s):
    """Minimal forward evaluations, forward pass included (checkpoint.py:129-135)."""
    if m < 1:
        raise ValidationError("need at least one step")
    if s < 1:
        raise ValidationError("snapshot budget must be >= 1 (s = 0 is unsupported)")
    return int(_tables(m, s - 1)[1][m, s - 1])


def plan_binomial(m, s):
    """Recomputation-optimal schedule for m steps and s slots (checkpoint.py:210-235)."""
    if m < 1:
        raise ValidationError("need at least one step")
    if s < 1:
        raise ValidationError("snapshot budget must be >= 1 (s = 0 is unsupported)")
    if m <= s:
        return plan_store_all(m)
    _, _, kb, kt = _tables(m, s - 1)
    acts = [Store(0, 0)]
    stores = {0: 0}
    free = list(range(s - 1, 0, -1))
    # explicit stack replaces the reference's mutual recursion; tasks run LIFO
    stack = [("total", 0, m, 0)]
    while stack:
        task = stack.pop()
        kind = task[0]
        if kind == "release":
            free.append(task[1])
            continue
        _, a, b, slot_a = task
        l = b - a
        if kind == "total":
            if l == 1:
                acts += [Advance(a, b), Restore(slot_a, a), AdjointStep(a)]
                continue
            k = int(kt[l, len(free)])
            if k < 0:
                acts.append(Advance(a, b))
                stack.append(("back", a, b, slot_a))
                continue
            mid = a + k
            slot = free.pop()
            acts += [Advance(a, mid), Store(slot, mid)]
            stores[mid] = slot
            stack += [("back", a, mid, slot_a), ("release", slot), ("total", mid, b, slot)]
        else:  # backward phase over [a, b), left state in slot_a
            if l == 0:
                continue
            if l == 1:
                acts += [Restore(slot_a, a), AdjointStep(a)]
                continue
            k = int(kb[l, len(free)])
            if k < 0:
                for n in range(b - 1, a, -1):
                    acts += [Restore(slot_a, a), Advance(a, n), AdjointStep(n)]
                acts += [Restore(slot_a, a), AdjointStep(a)]
                continue
            mid = a + k
            slot = free.pop()
            acts += [Restore(slot_a, a), Advance(a, mid), Store(slot, mid)]
            stack += [("back", a, mid, slot_a), ("release", slot), ("back", mid, b, slot)]
    acts.append(Done())
    start = 0
    for i, act in enumerate(acts):
        if isinstance(act, Advance) and act.stop == m:
            start = i + 1
            break
    return Schedule(n_steps=m, slots=s, actions=acts, recomputed=binomial_cost(m, s) - m,
                    forward_stores=stores, backward_start=start)


@dataclass
class SimReport:
    forward_evals: int
    max_live: int
    adjoint_steps: int


def simulate_schedule(schedule, step_oracle=None):
    """Replay a schedule against counters, enforcing its invariants (checkpoint.py:245-308)."""
    m = schedule.n_steps
    current, slots, max_live, evals, next_adj, done = 0, {}, 0, 0, m - 1, False
    for idx, act in enumerate(schedule.actions):
        if done:
            raise ScheduleError(f"action {idx}: actions after Done")
        if isinstance(act, Store):
            if current != act.step:
                raise ScheduleError(f"action {idx}: Store at step {act.step} but state is at {current}")
            slots[act.slot] = act.step
            if len(slots) > schedule.slots:
                raise ScheduleError(f"action {idx}: more than {schedule.slots} snapshots live")
            max_live = max(max_live, len(slots))
        elif isinstance(act, Restore):
            if act.slot not in slots:
                raise ScheduleError(f"action {idx}: Restore from empty slot {act.slot}")
            if slots[act.slot] != act.step:
                raise ScheduleError(f"action {idx}: slot {act.slot} holds step "
                                    f"{slots[act.slot]}, not {act.step}")
            current = act.step
        elif isinstance(act, Advance):
            if current != act.start:
                raise ScheduleError(f"action {idx}: Advance from {act.start} but state is at {current}")
            if not (act.start < act.stop <= m):
                raise ScheduleError(f"action {idx}: bad Advance range {act}")
            if step_oracle is not None:
                step_oracle(act.start, act.stop)
            evals += act.stop - act.start
            current = act.stop
        elif isinstance(act, AdjointStep):
            if act.step != next_adj:
                raise ScheduleError(f"action {idx}: AdjointStep({act.step}) out of order, "
                                    f"expected {next_adj}")
            if current != act.step:
                raise ScheduleError(f"action {idx}: AdjointStep({act.step}) but state is at {current}")
            next_adj -= 1
        elif isinstance(act, Done):
            done = True
        else:
            raise ScheduleError(f"action {idx}: unknown action {act!r}")
    if next_adj != -1:
        raise ScheduleError(f"incomplete schedule: next adjoint step {next_adj}")
    return SimReport(forward_evals=evals, max_live=max_live, adjoint_steps=m)
