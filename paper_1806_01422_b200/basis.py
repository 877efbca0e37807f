"""Host-side reference-element constants (GLL rule, D, element M/K).

These are computed once per operator on the host and shipped to the device as
kernel parameters.  They must be bit-identical to the reference
(``semopt/basis.py:48-154``) because every later tolerance is measured against
it; the arithmetic below therefore evaluates the same expressions in the same
association order with the same numpy primitives (checked bit-for-bit against
``tests/golden/basis.npz`` for N = 1..32, 48, 64).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NumericFailure, ValidationError

_TOL = 1e-14     # Newton tolerance, basis.py:19
_MAXIT = 100     # basis.py:20


@dataclass(frozen=True)
class SpectralBasis1D:
    degree: int
    nodes: np.ndarray
    weights: np.ndarray
    diff: np.ndarray


@dataclass(frozen=True)
class ElementOperators1D:
    length: float
    mass: np.ndarray
    stiffness: np.ndarray
    diff: np.ndarray


def legendre(degree, x):
    """(P_N(x), P_N'(x)) via Bonnet's recurrence and its derivative (basis.py:48-66)."""
    x = np.asarray(x, dtype=float)
    prev_p, prev_d = np.ones_like(x), np.zeros_like(x)
    if degree == 0:
        return prev_p, prev_d
    cur_p, cur_d = x.copy(), np.ones_like(x)
    for k in range(1, degree):
        nxt_p = ((2 * k + 1) * x * cur_p - k * prev_p) / (k + 1)
        nxt_d = ((2 * k + 1) * (cur_p + x * cur_d) - k * prev_d) / (k + 1)
        prev_p, cur_p = cur_p, nxt_p
        prev_d, cur_d = cur_d, nxt_d
    return cur_p, cur_d


def _interior_roots(n):
    """Roots of P_n' by damped Newton from Chebyshev-Lobatto points (basis.py:84-101)."""
    x = -np.cos(np.pi * np.arange(1, n) / n)
    half_gap = 0.5 * (np.pi / n)
    for _ in range(_MAXIT):
        p, dp = legendre(n, x)
        d2p = (2.0 * x * dp - n * (n + 1) * p) / (1.0 - x * x)
        dx = np.clip(dp / d2p, -half_gap, half_gap)
        x = x - dx
        if np.max(np.abs(dx)) <= _TOL:
            return x
    raise NumericFailure(f"GLL node iteration did not converge for degree {n}")


def gll_rule(degree):
    """GLL nodes/weights/D for one degree (basis.py:69-117)."""
    if not isinstance(degree, (int, np.integer)) or degree < 1:
        raise ValidationError(f"degree must be an integer >= 1, got {degree!r}")
    n = int(degree)
    xs = np.empty(n + 1)
    xs[0], xs[n] = -1.0, 1.0
    if n >= 2:
        xs[1:n] = _interior_roots(n)
    xs = 0.5 * (xs - xs[::-1])
    xs[0], xs[n] = -1.0, 1.0
    pn, _ = legendre(n, xs)
    w = 2.0 / (n * (n + 1) * pn * pn)
    w = 0.5 * (w + w[::-1])
    b = SpectralBasis1D(degree=n, nodes=xs, weights=w, diff=diff_matrix_from_nodes(xs))
    for a in (b.nodes, b.weights, b.diff):
        a.setflags(write=False)
    return b


def diff_matrix_from_nodes(nodes):
    """D[i, j] = l_j'(x_i); barycentric off-diagonal, negative-sum diagonal (basis.py:120-134)."""
    x = np.asarray(nodes, dtype=float)
    gaps = x[:, None] - x[None, :]
    np.fill_diagonal(gaps, 1.0)
    lam = 1.0 / np.prod(gaps, axis=1)
    d = (lam[None, :] / lam[:, None]) / gaps
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -np.sum(d, axis=1))
    return d


def diff_matrix(basis):
    return diff_matrix_from_nodes(basis.nodes)


def element_operators(basis, length):
    """M_e = (L/2) rho, K_e = sym((2/L) D^T diag(rho) D)  (basis.py:142-154)."""
    if not np.isfinite(length) or length <= 0.0:
        raise ValidationError(f"element length must be positive, got {length!r}")
    length = float(length)
    d = basis.diff
    k = (2.0 / length) * (d.T * basis.weights) @ d
    ops = ElementOperators1D(length=length, mass=(length / 2.0) * basis.weights,
                             stiffness=0.5 * (k + k.T), diff=d)
    ops.mass.setflags(write=False)
    ops.stiffness.setflags(write=False)
    return ops
