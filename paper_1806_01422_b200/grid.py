"""1D uniform GLL mesh metadata and assembly maps (reference ``semopt/grid.py``).

Design for the B200 path: the reference materialises an (E, N+1) int64
local->global table and (ndof,) multiplicity / mass / mask arrays
(``grid.py:65-72,112-146``) -- 2.15 GB of table alone at E = 2^25.  A uniform
1D mesh needs none of them: element e owns the contiguous node range
[e*N, e*N+N] (mod ndof when periodic), the mass diagonal is a per-local-index
pattern, and the Dirichlet mask touches two nodes.  The kernels use the
closed forms; the full arrays exist here only as lazily built host
properties so the reference's attribute surface (and the bit-exact tests
against it) keep working.

3D periodic boxes (``grid.py:113-122,239-244``) are :class:`Grid3D` (SURVEY.md
section 8(f) row 2); their operators live in ``ops3d.py``.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .basis import gll_rule
from .errors import ValidationError

PERIODIC = "periodic"
DIRICHLET0 = "dirichlet0"
SNAPSHOT_MAGIC = "semopt-field v1"    # grid.py:27


@dataclass(frozen=True)
class Axis:
    """Extent, element count, degree and boundary kind of the single axis."""

    xa: float
    xb: float
    elements: int
    degree: int
    bc: str = PERIODIC

    def __post_init__(self):
        # same admissibility rules as grid.py:40-50
        if self.xb <= self.xa:
            raise ValidationError(f"axis extent is empty: [{self.xa}, {self.xb}]")
        if self.elements < 1:
            raise ValidationError("need at least one element per axis")
        if self.degree < 1:
            raise ValidationError("polynomial degree must be >= 1")
        if self.bc not in (PERIODIC, DIRICHLET0):
            raise ValidationError(f"unknown boundary kind {self.bc!r}")
        if self.bc == PERIODIC and self.elements * self.degree < 2:
            raise ValidationError("periodic axis needs E*N >= 2 (degenerate wrap)")

    @property
    def length(self):
        return self.xb - self.xa

    @property
    def element_length(self):
        return (self.xb - self.xa) / self.elements

    @property
    def npts(self):
        return self.elements * self.degree + (0 if self.bc == PERIODIC else 1)

    def local_to_global(self):
        """(E, N+1) table e*N + i (mod npts if periodic) -- test/inspection only."""
        tab = (np.arange(self.elements)[:, None] * self.degree
               + np.arange(self.degree + 1)[None, :])
        return tab % self.npts if self.bc == PERIODIC else tab

    def coordinates(self):
        """Node coordinates, vectorised closed form of grid.py:74-84: each node takes
        the value written last by the reference loop (the right element at interfaces)."""
        xi = gll_rule(self.degree).nodes
        h, E, N = self.element_length, self.elements, self.degree
        left = self.xa + np.arange(E) * h
        loc = left[:, None] + h * (xi + 1.0) / 2.0
        out = np.empty(self.npts)
        out[:E * N] = loc[:, :N].ravel()
        if self.bc == PERIODIC:
            out[0] = self.xa
        else:
            out[E * N] = loc[E - 1, N]
        return out


class Grid:
    """1D mesh + assembly metadata.  Build through :func:`grid_1d`/:func:`build_grid`;
    ``Grid(axes)`` with three axes returns a :class:`Grid3D` (the reference's Grid serves
    both, grid.py:88-146)."""

    def __new__(cls, axes, element_length=None):
        axes = tuple(axes)
        if cls is Grid and len(axes) == 3:
            return Grid3D(axes)
        return super().__new__(cls)

    def __init__(self, axes, element_length=None):
        """``element_length`` overrides (xb - xa) / E: a shard of a larger mesh must use
        the global h bit for bit (K, M^-1 depend on it), whatever its local extent."""
        axes = tuple(axes)
        if len(axes) != 1:
            raise ValidationError(
                "only 1D grids are on the B200 hot path (3D sum-factorised grids are out of scope)")
        ax = axes[0]
        self.axes = axes
        self.axis = ax
        self.dim = 1
        self.ncomp = 1
        self.bases = (gll_rule(ax.degree),)
        self.shape = (ax.npts,)
        self.nscalar = ax.npts
        self.nglobal = ax.npts
        self.nelem = ax.elements
        self.local_shape = (ax.degree + 1,)
        self.periodic = ax.bc == PERIODIC
        self.has_mask = not self.periodic
        self.h = ax.element_length if element_length is None else float(element_length)
        # per-position mass pattern (see include/sem1d.h): [0] interface,
        # [1..N-1] interior, [N] first / [N+1] last node of a Dirichlet grid.
        # bincount sums (0 + a) + b at an interface (grid.py:157-161); a + b is
        # commutative, so every position is reproduced bit for bit.
        rho = self.bases[0].weights
        m_loc = (self.h / 2.0) * rho
        N = ax.degree
        pat = np.empty(N + 2)
        pat[1:N] = m_loc[1:N]
        if self.periodic or ax.elements > 1:
            pat[0] = m_loc[N] + m_loc[0]
        else:
            pat[0] = m_loc[0]
        pat[N] = m_loc[0]
        pat[N + 1] = m_loc[N]
        if N == 1 and self.periodic and ax.elements == 1:  # excluded by Axis, kept explicit
            raise ValidationError("degenerate periodic grid")
        self.mass_pattern = pat
        self.minv_pattern = 1.0 / pat   # ops.py:116 (1.0 / mass)
        if np.any(pat <= 0.0):
            raise ValidationError("assembled mass diagonal is not positive")

    # -- lazily materialised reference attributes (test / inspection only) --------

    @cached_property
    def table(self):
        t = np.ascontiguousarray(self.axis.local_to_global())
        t.setflags(write=False)
        return t

    def _expand(self, pat):
        E, N = self.axis.elements, self.axis.degree
        out = np.empty(self.nglobal)
        out[:E * N] = np.tile(pat[:N], E)
        if not self.periodic:
            out[0] = pat[N]
            out[E * N] = pat[N + 1]
        out.setflags(write=False)
        return out

    @cached_property
    def mass_scalar(self):
        return self._expand(self.mass_pattern)

    @cached_property
    def multiplicity(self):
        E, N = self.axis.elements, self.axis.degree
        pat = np.ones(N + 2)
        pat[0] = 2.0 if (self.periodic or E > 1) else 1.0
        return self._expand(pat)

    @cached_property
    def mask_scalar(self):
        m = np.ones(self.nglobal)
        if not self.periodic:
            m[0] = 0.0
            m[-1] = 0.0
        m.setflags(write=False)
        return m

    # -- maps on device fields (C ABI) ------------------------------------------

    def scatter(self, u):
        """Global -> (1, E, N+1) element copies (grid.py:165-169), on the device."""
        from . import ops
        return ops._grid_scatter(self, u)

    def gather(self, local):
        """Adjoint of scatter (grid.py:171-182), on the device."""
        from . import ops
        return ops._grid_gather(self, local)

    def mask(self, u):
        """Zero the Dirichlet end nodes (grid.py:184-189); works on numpy or torch."""
        if not self.has_mask:
            return u
        if isinstance(u, np.ndarray):
            self._check_host(u)
            return u * self.mask_scalar
        out = u.clone()
        out[..., 0] = out[..., 0] * 0.0
        out[..., -1] = out[..., -1] * 0.0
        return out

    def mass(self):
        return self.mass_scalar

    def _check_host(self, u):
        u = np.asarray(u, dtype=float)
        if u.shape != (self.nglobal,):
            raise ValidationError(f"field has shape {u.shape}, expected ({self.nglobal},)")
        return u

    # -- geometry -------------------------------------------------------------

    def node_coordinates(self):
        return (self.axis.coordinates(),)

    def evaluate(self, fn):
        """Sample x -> fn(x) at the nodes, masked (grid.py:209-222)."""
        vals = np.asarray(fn(self.node_coordinates()[0]), dtype=float).ravel()
        return self.mask(vals)

    def l2_norm(self, u):
        """sqrt(u^T M u) (grid.py:224-227)."""
        if isinstance(u, np.ndarray):
            u = self._check_host(u)
            return float(np.sqrt(np.dot(u, self.mass_scalar * u)))
        import torch
        m = torch.as_tensor(self.mass_scalar, device=u.device)
        return float(torch.sqrt(torch.dot(u, m * u)))


class Grid3D:
    """Periodic 3D box with a 3-component field (reference Grid with three axes,
    grid.py:112-146).  One degree on all axes (the kernels' constraint); extents and
    element counts may differ per axis.  The assembly maps are closed forms on the
    device; the reference's tables / bincount masses exist here only as lazily built
    host arrays for inspection and the bit-exact tests."""

    def __init__(self, axes):
        axes = tuple(axes)
        if len(axes) != 3:
            raise ValidationError("Grid3D needs three axes")
        if any(ax.bc != PERIODIC for ax in axes):
            raise ValidationError("unsupported configuration: 3D grids require periodic axes")
        if len({ax.degree for ax in axes}) != 1:
            raise ValidationError("the B200 3D kernels need the same degree on every axis")
        self.axes = axes
        self.dim = 3
        self.ncomp = 3
        self.N = axes[0].degree
        self.bases = tuple(gll_rule(ax.degree) for ax in axes)
        self.shape = tuple(ax.npts for ax in axes)
        self.nscalar = int(np.prod(self.shape))
        self.nglobal = 3 * self.nscalar
        self.nelem = int(np.prod([ax.elements for ax in axes]))
        self.local_shape = (self.N + 1,) * 3
        self.periodic = True
        self.has_mask = False
        self.h = tuple(ax.element_length for ax in axes)
        self.mvec = tuple((ax.element_length / 2.0) * b.weights for ax, b in zip(axes, self.bases))
        self.mass_pattern = self._mass_pattern()
        self.minv_pattern = 1.0 / self.mass_pattern

    # bincount of the element mass blocks in table order (grid.py:131-135, 150-161) on a
    # box of min(E_a, 2) elements per axis: it holds every position class (interior node,
    # wrap node g = 0, other interface) with the same per-node summation order
    def _mass_pattern(self):
        N, n = self.N, self.N + 1
        Es = [min(ax.elements, 2) for ax in self.axes]
        Ps = [E * N for E in Es]
        tabs = [((np.arange(E)[:, None] * N + np.arange(n)[None, :]) % P) for E, P in zip(Es, Ps)]
        g1 = tabs[0][:, None, None, :, None, None]
        g2 = tabs[1][None, :, None, None, :, None]
        g3 = tabs[2][None, None, :, None, None, :]
        table = ((g1 * Ps[1] + g2) * Ps[2] + g3).reshape(-1)
        m1, m2, m3 = self.mvec
        blk = m1[:, None, None] * m2[None, :, None] * m3[None, None, :]
        ne = int(np.prod(Es))
        mass = np.bincount(table, weights=np.broadcast_to(blk, (ne, n, n, n)).ravel(),
                           minlength=int(np.prod(Ps))).reshape(Ps)
        pat = np.empty((N + 1,) * 3)
        pos = [[0] + list(range(1, N)) + [N if E > 1 else 0] for E in Es]   # class -> node
        for c1 in range(N + 1):
            for c2 in range(N + 1):
                for c3 in range(N + 1):
                    pat[c1, c2, c3] = mass[pos[0][c1], pos[1][c2], pos[2][c3]]
        return pat.ravel()

    # -- lazily materialised reference attributes (inspection / tests) ------------

    @cached_property
    def table(self):
        N, n = self.N, self.N + 1
        tabs = [ax.local_to_global() for ax in self.axes]
        n2, n3 = self.shape[1], self.shape[2]
        g1 = tabs[0][:, None, None, :, None, None]
        g2 = tabs[1][None, :, None, None, :, None]
        g3 = tabs[2][None, None, :, None, None, :]
        t = np.ascontiguousarray(((g1 * n2 + g2) * n3 + g3).reshape(self.nelem, n, n, n))
        t.setflags(write=False)
        return t

    @cached_property
    def mass_scalar(self):
        """The assembled mass diagonal by position class (bit-identical to the reference's
        bincount, tests/test_host.py)."""
        N = self.N
        cls = []
        for P in self.shape:
            g = np.arange(P)
            r = g % N
            cls.append(np.where(r != 0, r, np.where(g == 0, 0, N)))
        idx = (cls[0][:, None, None] * (N + 1) + cls[1][None, :, None]) * (N + 1) + cls[2][None, None, :]
        m = self.mass_pattern[idx].ravel()
        m.setflags(write=False)
        return m

    def mass(self):
        return np.tile(self.mass_scalar, 3)

    def mask(self, u):
        return u                                   # periodic boxes only

    def scatter(self, u):
        """Global -> (3, nelem, n, n, n) element blocks (grid.py:165-169), host arrays."""
        u = self._check_host(u)
        return u.reshape(3, self.nscalar)[:, self.table]

    def gather(self, local):
        """Adjoint of scatter (grid.py:171-182), host arrays."""
        out = np.empty(self.nglobal)
        for c in range(3):
            out[c * self.nscalar:(c + 1) * self.nscalar] = np.bincount(
                self.table.ravel(), weights=np.ascontiguousarray(local[c]).ravel(), minlength=self.nscalar)
        return out

    def _check_host(self, u):
        u = np.asarray(u, dtype=float)
        if u.shape != (self.nglobal,):
            raise ValidationError(f"field has shape {u.shape}, expected ({self.nglobal},)")
        return u

    def node_coordinates(self):
        return tuple(ax.coordinates() for ax in self.axes)

    def evaluate(self, fn):
        """(x1, x2, x3) meshes -> 3 component arrays (grid.py:209-222)."""
        mesh = np.meshgrid(*self.node_coordinates(), indexing="ij")
        comps = fn(*mesh)
        return np.concatenate([np.asarray(c, dtype=float).ravel() for c in comps])

    def l2_norm(self, u):
        if isinstance(u, np.ndarray):
            u = self._check_host(u)
            return float(np.sqrt(np.dot(u, self.mass() * u)))
        import torch
        m = torch.as_tensor(self.mass(), device=u.device)
        return float(torch.sqrt(torch.dot(u, m * u)))


def build_grid(axes):
    axes = tuple(axes)
    return Grid3D(axes) if len(axes) == 3 else Grid(axes)


def grid_1d(xa, xb, elements, degree, bc=PERIODIC):
    return Grid([Axis(xa, xb, elements, degree, bc)])


def grid_3d(extents, elements, degree):
    """Periodic 3D box (grid.py:239-244); extents is ((xa, xb),)*3 or one (xa, xb) pair."""
    if len(extents) == 2 and np.isscalar(extents[0]):
        extents = (extents,) * 3
    return Grid3D([Axis(e[0], e[1], elements, degree, PERIODIC) for e in extents])


# -- field snapshots (reference grid.py:250-305) ---------------------------------
#
# Format: an ASCII header (magic line, "dim", "ncomp", one "axis" line per axis with
# elements / degree / repr'd extent / bc, "count", "end-header"), then `count`
# little-endian float64 values.  Files written here are byte-identical to the
# reference's for the same grid and values, and either side reads the other's.


def _host_values(grid, values):
    """Field -> contiguous host float64 array of shape (nglobal,) (device tensors copied)."""
    if not isinstance(values, np.ndarray) and hasattr(values, "detach"):
        values = values.detach().cpu().numpy()
    v = np.asarray(values, dtype=float)
    if v.shape != (grid.nglobal,):
        raise ValidationError(f"field has shape {v.shape}, expected ({grid.nglobal},)")
    return v


def save_field(path, grid, values):
    """Write a field snapshot (grid.py:253-270)."""
    v = _host_values(grid, values)
    lines = [SNAPSHOT_MAGIC, f"dim {grid.dim}", f"ncomp {grid.ncomp}"]
    for k, ax in enumerate(grid.axes):
        lines.append(f"axis {k} elements {ax.elements} degree {ax.degree} "
                     f"extent {ax.xa!r} {ax.xb!r} bc {ax.bc}")
    lines += [f"count {grid.nglobal}", "end-header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(lines) + "\n").encode("ascii"))
        fh.write(v.astype("<f8", copy=False).tobytes())


def load_field(path):
    """Read a snapshot (grid.py:273-305); returns (grid, values).  3D snapshots parse but
    their grid is outside the B200 path (ValidationError from Grid)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    marker = b"end-header\n"
    cut = blob.find(marker)
    if cut < 0 or not blob.startswith(SNAPSHOT_MAGIC.encode("ascii")):
        raise ValidationError(f"{path}: not a semopt field snapshot")
    meta, axes_kv = {}, {}
    for line in blob[:cut].decode("ascii").splitlines()[1:]:
        parts = line.split()
        if not parts:
            continue
        if parts[0] == "axis":
            axes_kv[int(parts[1])] = parts[2:]
        else:
            meta[parts[0]] = parts[1:]
    try:
        dim, count = int(meta["dim"][0]), int(meta["count"][0])
        axes = []
        for k in range(dim):
            f = axes_kv[k]
            ext = f.index("extent")
            axes.append(Axis(xa=float(f[ext + 1]), xb=float(f[ext + 2]),
                             elements=int(f[f.index("elements") + 1]),
                             degree=int(f[f.index("degree") + 1]), bc=f[f.index("bc") + 1]))
    except (KeyError, ValueError, IndexError) as exc:
        raise ValidationError(f"{path}: malformed snapshot header ({exc})") from exc
    grid = Grid(axes)
    if grid.nglobal != count:
        raise ValidationError(f"{path}: header count {count} != grid {grid.nglobal}")
    payload = blob[cut + len(marker):]
    if len(payload) < 8 * count:
        raise ValidationError(f"{path}: payload holds {len(payload) // 8} values, header says {count}")
    return grid, np.frombuffer(payload, dtype="<f8", count=count).astype(float)
