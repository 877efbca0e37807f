"""Element-sharded operator for multi-GPU runs (BASELINE config 5).

Partition: rank r of P owns the contiguous element block [e_lo, e_hi) and the
global nodes [e_lo*N, e_hi*N) (plus node E*N on the last rank of a Dirichlet
grid).  Each rank stores its fields on an EXTENDED chain: its elements plus
one ghost element on each side that has a neighbour (no ghost at a global
Dirichlet end; two on the left, see Partition), laid out as a local Dirichlet grid with the GLOBAL element
length h.  On periodic global rings each rank instead keeps ghost ZONES of 8
elements per side on a periodic local chain, so the single-launch RK step and
adjoint step kernels run after ONE exchange per step (Partition docstring).  The unchanged fused kernels then compute, on every rank, both
contributions to each owned interface node -- including node e_lo*N, whose
left contribution comes from the recomputed ghost element -- so a sharded
apply is bit-identical to the single-GPU apply (the interface sum has the same
two terms; K and M^-1 are built from the same h).

Communication per operator input: one ghost refresh -- send the first N+1
owned nodes to the left neighbour and the last 2N owned nodes to the right
neighbour (torch.distributed P2P: NCCL over NVLink on GPUs, gloo on CPU for
the tests).  Dot products (the objective, L-BFGS) all-reduce the owned parts.
The stage kernels run unchanged on extended fields; before each stage the
inputs the kernel reads across element boundaries (U, and lam / l_j for the
adjoint) are refreshed in one batched exchange.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ValidationError
from .grid import DIRICHLET0, PERIODIC, Axis, Grid


class Partition:
    """Contiguous element blocks; ghost elements where a neighbour exists.

    ``zone`` = 0: the minimal Dirichlet-chain layout (2 ghost elements left, 1 right).
    ``zone`` = G > 0 (periodic global rings only): G ghost elements on each side and the
    extended chain is itself treated as a PERIODIC ring -- the wrap-around garbage of a
    step reaches at most 2s-1 elements into the chain, i.e. stays in the ghost zone when
    G >= 2s-1, so the single-launch step kernels run unchanged after one exchange."""

    def __init__(self, E, N, P, rank, periodic, zone=0):
        if P < 1 or not (0 <= rank < P):
            raise ValidationError(f"bad rank {rank} of {P}")
        if E < 3 * P:
            raise ValidationError(f"need at least 3 elements per rank (E={E}, P={P})")
        if zone and not periodic:
            raise ValidationError("ghost zones need a periodic global ring")
        self.zone = int(zone) if P > 1 else 0
        self.E, self.N, self.P, self.rank, self.periodic = E, N, P, rank, bool(periodic)
        self.e_lo = (rank * E) // P
        self.e_hi = ((rank + 1) * E) // P
        self.E_loc = self.e_hi - self.e_lo
        last_dirichlet = (not self.periodic) and rank == P - 1
        self.n_own = self.E_loc * N + (1 if last_dirichlet else 0)
        # two ghost elements on the left: J^T masks and M^-1-scales its INPUT at the
        # chain's end node (ops.py:252-254), so element e_lo-1 (which contributes to the
        # owned node e_lo*N) must not touch the chain end; one on the right suffices
        # because node e_hi*N is not owned.
        self.gl = 2 if (self.periodic or rank > 0) else 0
        self.gr = 1 if (self.periodic or rank < P - 1) else 0
        if self.zone:
            if self.E_loc < self.zone:
                raise ValidationError(f"ghost zone {self.zone} exceeds the {self.E_loc}-element block")
            self.gl = self.gr = self.zone
        if P == 1:
            self.gl = self.gr = 0
        self.E_ext = self.E_loc + self.gl + self.gr
        self.own0 = self.gl * N                       # owned range start in the ext chain
        self.ext_ndof = self.E_ext * N + (0 if self.zone else 1)
        self.left = (rank - 1) % P if self.gl else None
        self.right = (rank + 1) % P if self.gr else None
        self.g_lo = self.e_lo * N                     # global index of the first owned node

    def owned_slice(self):
        return slice(self.own0, self.own0 + self.n_own)


class HaloExchange:
    """Ghost refresh of extended fields through torch.distributed point-to-point ops."""

    def __init__(self, part, group=None):
        self.p, self.group = part, group

    def refresh(self, fields):
        """Fill the ghost nodes of every extended field in ``fields``: one batched P2P round
        whose messages go straight from each field's owned edge slice into the neighbour's
        ghost slice (contiguous views, no pack / unpack kernels)."""
        self.start(fields).finish()

    class _Pending:
        def __init__(self, works=(), copies=()):
            self.works, self.copies = list(works), list(copies)

        def finish(self):
            """NCCL: the current stream waits for the exchange (no host sync); gloo: the
            staged receives land in the ghost slices."""
            for r in self.works:
                r.wait()
            for dst, src in self.copies:
                dst.copy_(src)
            self.works, self.copies = [], []

    def start(self, fields):
        """Post the exchange of ``fields`` and return a handle whose ``finish()`` makes the
        current stream wait for it: kernels launched in between (the interior tiles of a
        step, which read no ghost node) overlap the transfer."""
        import torch
        import torch.distributed as dist
        p = self.p
        if p.P == 1 or not fields:
            return self._Pending()
        N = p.N
        o0, no = p.own0, p.n_own
        L = p.gl * N                       # left ghost nodes I receive
        R = p.gr * N + (0 if p.zone else 1)  # right ghost nodes I receive
        # what the neighbours receive from me: every rank that has a left (right)
        # neighbour has the same left (right) ghost width -- 2N (N+1) for Dirichlet chains,
        # zone*N in ghost-zone mode -- so the sizes are the neighbours', not mine
        to_left = p.zone * N if p.zone else N + 1
        to_right = p.zone * N if p.zone else 2 * N
        # per field: send left, send right, receive right, receive left.  NCCL pairs the
        # messages between two ranks in issue order (also when left and right neighbour are
        # the same rank, P = 2); gloo pairs them by tag (2i: sent leftwards, 2i+1: rightwards)
        ops, recvs = [], []
        for i, f in enumerate(fields):
            if p.left is not None:
                ops.append(dist.P2POp(dist.isend, f[o0:o0 + to_left], p.left, self.group, tag=2 * i))
            if p.right is not None:
                ops.append(dist.P2POp(dist.isend, f[o0 + no - to_right:o0 + no], p.right, self.group,
                                      tag=2 * i + 1))
            if p.right is not None:
                dst = f[o0 + no:o0 + no + R]
                ops.append(dist.P2POp(dist.irecv, dst, p.right, self.group, tag=2 * i))
                recvs.append(dst)
            if p.left is not None:
                dst = f[0:L]
                ops.append(dist.P2POp(dist.irecv, dst, p.left, self.group, tag=2 * i + 1))
                recvs.append(dst)
        staged = fields[0].device.type == "cuda" and dist.get_backend(self.group) == "gloo"
        if staged:   # gloo moves CPU tensors only: stage through host memory
            ops = [dist.P2POp(o.op, o.tensor.cpu() if o.op is dist.isend else
                              torch.empty(o.tensor.shape, dtype=o.tensor.dtype), o.peer, self.group,
                              tag=o.tag) for o in ops]
            recv_cpu = [o.tensor for o in ops if o.op is dist.irecv]
        works = dist.batch_isend_irecv(ops)
        if staged:                    # host-side transfers: complete them now
            for r in works:
                r.wait()
            return self._Pending(copies=list(zip(recvs, recv_cpu)))
        return self._Pending(works=works)


def shard_grid(global_grid, part):
    """The extended local chain of a partition with the global h: a Dirichlet chain, or a
    periodic one in ghost-zone mode (a single rank keeps the global grid itself)."""
    if part.P == 1:
        return global_grid
    ax = global_grid.axis
    h = global_grid.h
    xa = ax.xa + (part.e_lo - part.gl) * h
    xb = xa + part.E_ext * h
    bc = PERIODIC if part.zone else DIRICHLET0
    return Grid([Axis(xa, xb, part.E_ext, ax.degree, bc)], element_length=h)


class ShardedOperator:
    """Drop-in for ``SemOperator`` on one rank of an element-sharded grid.

    Fields are EXTENDED tensors (``ext_ndof`` entries, ghost nodes included);
    ``field()`` accepts either the owned part (``n_own``) or an extended tensor,
    ``public()`` returns the owned part.  ``local_factory(grid, coef)`` builds the
    rank-local operator (the CUDA SemOperator by default; the CPU tests pass a
    test double with the same launch interface)."""

    def __init__(self, global_grid, coef, rank, world, group=None, local_factory=None, device=None,
                 zone=None):
        self.global_grid = global_grid
        self.coef = coef
        if zone is None:   # periodic rings: ghost zones wide enough for a fused RK4 adjoint step
            zone = 8 if global_grid.periodic else 0
        self.part = Partition(global_grid.axis.elements, global_grid.axis.degree, world, rank,
                              global_grid.periodic, zone=zone)
        self.grid = shard_grid(global_grid, self.part)
        if local_factory is None:
            from .ops import SemOperator

            def local_factory(g, c):
                return SemOperator(g, c, device=device)
        self.local = local_factory(self.grid, coef)
        self.device = self.local.device
        self.batch = 1
        self.ndof = self.part.ext_ndof
        self.shape = (self.ndof,)
        self.halo = HaloExchange(self.part, group)
        self.group = group
        self.counters = self.local.counters
        self.sync_checks = True
        self.last_sweep_stats = {}
        self.max_matrix_dim = self.local.max_matrix_dim
        # owned-node mass pattern for the objective (global positions)
        m = global_grid.mass_pattern
        N = self.part.N
        g = self.part.g_lo + np.arange(self.part.n_own)
        pos = g % N
        mass = m[pos].copy()
        if not global_grid.periodic:
            mass[g == 0] = m[N]
            mass[g == global_grid.axis.elements * N] = m[N + 1]
        import torch
        self._mass_own = torch.as_tensor(mass, device=self.device)
        mask = np.ones(self.part.n_own)
        if not global_grid.periodic:
            mask[g == 0] = 0.0
            mask[g == global_grid.axis.elements * N] = 0.0
        self._mask_own = torch.as_tensor(mask, device=self.device)

    # -- fields -------------------------------------------------------------

    def empty(self):
        import torch
        return torch.zeros(self.shape, dtype=torch.float64, device=self.device)

    def field(self, x, name="field"):
        import torch
        host = not isinstance(x, torch.Tensor)
        t = torch.as_tensor(np.asarray(x, dtype=np.float64) if host else x)
        if t.dtype != torch.float64:
            raise ValidationError(f"{name} must be float64, got {t.dtype}")
        t = t.to(self.device)
        if tuple(t.shape) == (self.part.n_own,):
            e = self.empty()
            e[self.part.owned_slice()] = t
            self.halo.refresh([e])
            return e, host
        if tuple(t.shape) == self.shape:
            return t.contiguous(), host
        raise ValidationError(f"{name} has shape {tuple(t.shape)}, expected ({self.part.n_own},) "
                              f"owned or {self.shape} extended")

    def public(self, t):
        return t[self.part.owned_slice()]

    def _isfinite_all(self, t):
        import torch
        ok = torch.tensor([0.0 if bool(torch.isfinite(self.public(t)).all()) else 1.0],
                          device=self.device)
        self._allreduce(ok, "max")
        return float(ok.item()) == 0.0

    def _allreduce(self, t, op="sum"):
        import torch.distributed as dist
        if self.part.P > 1:
            rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
            if t.is_cuda and dist.get_backend(self.group) == "gloo":
                c = t.cpu()
                dist.all_reduce(c, op=rop, group=self.group)
                t.copy_(c)
            else:
                dist.all_reduce(t, op=rop, group=self.group)
        return t

    def flags(self, reset=True):
        """Device flags OR-ed over ranks, so every rank raises the same exception."""
        import torch
        v = self.local.flags(reset=reset)
        t = torch.tensor([float(v)], device=self.device)
        if self.part.P > 1:
            bits = torch.tensor([float(v & b) > 0 for b in (1, 2, 4)], dtype=torch.float64,
                                device=self.device)
            self._allreduce(bits, "max")
            v = sum(b for b, on in zip((1, 2, 4), bits.tolist()) if on)
        del t
        return int(v)

    def dot(self, a, b):
        """Global inner product of extended (or owned) fields: owned parts, all-reduced."""
        import torch
        a = self.public(a) if a.shape[-1] == self.ndof else a
        b = self.public(b) if b.shape[-1] == self.ndof else b
        t = torch.dot(a.reshape(-1), b.reshape(-1)).reshape(1)
        return float(self._allreduce(t, "sum").item())

    # -- launches: refresh what the kernel reads across element boundaries ------

    def refresh(self, fields):
        """One batched ghost exchange for several extended fields; launches on them may then
        pass refresh=False (e.g. a step applying F(u), J(u)v and J(u)^T w exchanges u, v and w
        once instead of once per apply)."""
        self.halo.refresh(list(fields))

    def launch_rhs(self, u, out, refresh=True):
        if refresh:
            self.halo.refresh([u])
        self.local.launch_rhs(u, out)

    def launch_jac(self, u, v, out, refresh=True):
        if refresh:
            self.halo.refresh([u, v])
        self.local.launch_jac(u, v, out)

    def launch_jact(self, u, z, out, refresh=True):
        if refresh:
            self.halo.refresh([u, z])
        self.local.launch_jact(u, z, out)

    def launch_rk_stage(self, U_in, k_out, base, terms, coefs, dt, Y, check):
        self.halo.refresh([U_in])
        self.local.launch_rk_stage(U_in, k_out, base, terms, coefs, dt, Y, check)

    def launch_adj_stage(self, U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out):
        self.halo.refresh([U, lam] + list(l_terms))
        self.local.launch_adj_stage(U, lam, b, l_terms, a_coefs, dt, l_out, acc_terms, lam_out)

    # -- whole-step launches (ghost-zone mode): one exchange per step ----------------

    def step_fused_supported(self):
        f = getattr(self.local, "step_fused_supported", None)
        return bool(self.part.zone >= 7 and f is not None and f())

    def _tile_split(self, kind, scheme):
        """(interior, edge) tile ranges (first, count) of a whole-step launch on the extended
        chain: interior tiles read no ghost element, so they run while the exchange is in
        flight (None: no split -- not the N = 7 kernels, or too few tiles)."""
        key = (kind, scheme)
        cache = self.__dict__.setdefault("_splits", {})
        if key in cache:
            return cache[key]
        split = None
        f = getattr(self.local, "step_tiling", None)
        if f is not None and self.part.zone and self.part.N == 7 and getattr(self, "overlap", True):
            try:
                nt, T, H = f(kind, False, scheme)
            except Exception:
                nt = 0
            z, Ee = self.part.zone, self.part.E_ext
            inner = [t for t in range(nt) if t * T - H >= z and (t + 1) * T + H <= Ee - z]
            if inner and inner == list(range(inner[0], inner[-1] + 1)) and len(inner) < nt:
                ta, tb = inner[0], inner[-1] + 1
                split = ((ta, tb - ta), (tb % nt, nt - tb + ta))
        cache[key] = split
        return split

    def launch_rk_step(self, u, u_new, dt, scheme, flag=None):
        kw = {} if flag is None else {"flag": flag}
        split = self._tile_split(0, scheme)
        if split is None:
            self.halo.refresh([u])
            self.local.launch_rk_step(u, u_new, dt, scheme, **kw)
            return
        pending = self.halo.start([u])          # ghosts of u in flight ...
        self.local.launch_rk_step(u, u_new, dt, scheme, tiles=split[0], **kw)   # ... interior tiles
        pending.finish()
        self.local.launch_rk_step(u, u_new, dt, scheme, tiles=split[1], **kw)   # edge tiles

    # run-ahead integrate (timeloop.integrate): per-step flag words of the local operator,
    # verified with one all-reduce per window so every rank rolls back at the same step
    @property
    def supports_flag_slots(self):
        return bool(getattr(self.local, "supports_flag_slots", False))

    def flag_slots(self, k):
        return self.local.flag_slots(k)

    def reduce_flag_words(self, words):
        """Bitwise OR over ranks of the window's flag words: each bit plane is all-reduced with
        MAX, so every rank sees the same failing step and the same failure kind."""
        import torch
        planes = torch.stack([(words & b) != 0 for b in (1, 2, 4)]).to(torch.float64)
        planes = self._allreduce(planes, "max")
        out = torch.zeros_like(words)
        for k, b in enumerate((1, 2, 4)):
            out |= (planes[k] > 0).to(words.dtype) * b
        return out

    def launch_adj_step(self, u, lam, lam_out, dt, scheme, flag=None):
        kw = {} if flag is None else {"flag": flag}
        split = self._tile_split(1, scheme)
        if split is None:
            self.halo.refresh([u, lam])
            self.local.launch_adj_step(u, lam, lam_out, dt, scheme, **kw)
            return
        pending = self.halo.start([u, lam])
        self.local.launch_adj_step(u, lam, lam_out, dt, scheme, tiles=split[0], **kw)
        pending.finish()
        self.local.launch_adj_step(u, lam, lam_out, dt, scheme, tiles=split[1], **kw)

    def launch_terminal(self, uN, ud, lam, J_out):
        """Objective on owned nodes, all-reduced; lam = mask(2 M d) (adjoint.py:39-47)."""
        sl = self.part.owned_slice()
        d = uN[sl] - ud[sl]
        md = self._mass_own * d
        lam.zero_()
        lam[sl] = (2.0 * md) * self._mask_own
        j = (d * md).sum().reshape(1)
        J_out.copy_(self._allreduce(j, "sum"))

    # -- reference surface ----------------------------------------------------

    def apply_rhs(self, u):
        ut, host = self.field(u, "state")
        self.counters["rhs"] += 1
        out = self.empty()
        self.launch_rhs(ut, out)
        self._raise(("state", "state"))
        return self._ret(out, host)

    def apply_jacobian(self, u, w):
        ut, host = self.field(u, "state")
        wt, _ = self.field(w, "tangent")
        self.counters["jac"] += 1
        out = self.empty()
        self.launch_jac(ut, wt, out)
        self._raise(("state", "tangent"))
        return self._ret(out, host)

    def apply_jacobian_transpose(self, u, z):
        ut, host = self.field(u, "state")
        zt, _ = self.field(z, "cotangent")
        self.counters["jact"] += 1
        out = self.empty()
        self.launch_jact(ut, zt, out)
        self._raise(("state", "cotangent"))
        return self._ret(out, host)

    def _raise(self, names):
        from .errors import NumericFailure
        v = self.flags()
        if v & _lib.SEM1D_FLAG_STATE_NONFINITE:
            raise NumericFailure(f"{names[0]} contains NaN/Inf")
        if v & _lib.SEM1D_FLAG_INPUT2_NONFINITE:
            raise NumericFailure(f"{names[1]} contains NaN/Inf")

    def _ret(self, t, host):
        o = self.public(t)
        return o.cpu().numpy() if host else o


def sharded_dot(op):
    """The ``dot`` callable for :func:`optimize.minimize` on sharded fields."""
    return op.dot


def init_from_env(backend=None):
    """torch.distributed init from torchrun's environment (MASTER_ADDR must be 127.0.0.1
    on these boxes).  Returns (rank, world, local_rank)."""
    import os

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return rank, world, local


__all__ = ["HaloExchange", "Partition", "ShardedOperator", "init_from_env", "shard_grid",
           "sharded_dot", "PERIODIC"]
