"""The BASELINE.json workloads as builders.

Inputs are seeded numpy PCG64 draws per global node in node order, created on
the host and shared unchanged by the oracle (tests / bench CPU leg) and the
device path.
"""

from __future__ import annotations

import numpy as np

from . import timeloop
from .grid import DIRICHLET0, PERIODIC, grid_1d
from .ops import PdeCoefficients, SemOperator
from .problems import AssimilationProblem

CFG1 = dict(xa=-1.0, xb=1.0, E=16, N=9, nu=0.01, steps=20, dt=1e-4, seed=1806)
CFG2 = dict(xa=-1.0, xb=1.0, E=1 << 22, N=7, nu=0.01, seed=2)
CFG3 = dict(xa=-1.0, xb=1.0, E=1 << 18, N=31, nu=1e-3, seed=3)
# config 4: dt = 5e-5 is unstable on [-1, 1] (rho(J) = 3.85e6, SURVEY.md finding 4);
# [0, 20] gives rho = 3.85e4 and an RK4 limit of ~7e-5.
CFG4 = dict(xa=0.0, xb=20.0, B=4096, E=256, N=15, nu=0.01, steps=1000, dt=5e-5, seed=4)
# config 5 gives neither domain nor dt: h = 1/64 (domain length 2^25 / 64) gives
# rho(J) ~ 5.4e3 at nu = 1e-3, N = 7 (oracle dense Jacobian at the same h), so RK4 is
# stable to dt ~ 5e-4; dt = 2e-4, 500 steps.  Binomial checkpointing with s = 40 slots
# (75 GB of 1.88 GB states on one 180 GB B200, leaving room for the L-BFGS vectors).
CFG5 = dict(h=1.0 / 64.0, E=1 << 25, N=7, nu=1e-3, steps=500, dt=2e-4, slots=40, modes=32,
            seed=5, lbfgs_iters=10)


def cfg1_inputs(grid, seed=CFG1["seed"]):
    """u0 = sin(pi x) + 0.01 N(0,1); target IC = sin(pi x) + 0.5 sin(2 pi x) (BASELINE config 1)."""
    x = grid.node_coordinates()[0]
    rng = np.random.default_rng(seed)
    u0 = grid.mask(np.sin(np.pi * x) + 0.01 * rng.standard_normal(grid.nglobal))
    obs0 = grid.mask(np.sin(np.pi * x) + 0.5 * np.sin(2.0 * np.pi * x))
    return u0, obs0


def cfg1_problem(bc=PERIODIC, scheme="rk4", checkpoint_slots=None, device=None, target=None):
    c = CFG1
    grid = grid_1d(c["xa"], c["xb"], c["E"], c["N"], bc)
    op = SemOperator(grid, PdeCoefficients(c["nu"]), device=device)
    ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=c["steps"] * c["dt"], dt=c["dt"])
    u0, obs0 = cfg1_inputs(grid)
    if target is None:
        target = timeloop.integrate(op, obs0, ts, store_steps=None).u_final
    return AssimilationProblem(name=f"cfg1-{bc}-{scheme}", grid=grid, op=op, ts=ts,
                               u_target=target, u_guess=u0, checkpoint_slots=checkpoint_slots)


def operator_inputs(ndof, seed):
    """u ~ U(-1,1), v ~ N(0,1), w ~ N(0,1) per node (BASELINE configs 2/3)."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, ndof)
    v = rng.standard_normal(ndof)
    w = rng.standard_normal(ndof)
    return u, v, w


def fourier_fields(grid, batch, n_modes, seed):
    """Per problem: sum_k a_k sin(2 pi k (x - xa) / L), a_k ~ U(-1, 1) (BASELINE configs 4/5)."""
    ax = grid.axis
    x = grid.node_coordinates()[0]
    rng = np.random.default_rng(seed)
    amps = rng.uniform(-1.0, 1.0, (batch, n_modes))
    k = np.arange(1, n_modes + 1)
    phase = 2.0 * np.pi * np.outer(k, (x - ax.xa) / ax.length)   # (modes, ndof)
    return amps @ np.sin(phase)


def fourier_field_device(grid, n_modes, seed, device, band=None):
    """One seeded smooth Fourier field sum_k a_k sin(2 pi k (x - xa) / L), a_k ~ U(-1, 1),
    evaluated on the device from the closed-form node coordinates (config 5 sizes make
    the host outer product of fourier_fields prohibitive).  ``band`` = (kmin, kmax): the n_modes
    angular wavenumbers are drawn uniformly from that band instead (rounded to periodic
    modes of the ring), so the fields have structure on the element scale, where viscosity
    acts within a config-5 horizon."""
    import torch
    ax = grid.axis
    rng = np.random.default_rng(seed)
    amps = rng.uniform(-1.0, 1.0, n_modes)
    if band is not None:
        kappa = rng.uniform(band[0], band[1], n_modes)
        modes = np.maximum(1.0, np.round(kappa * ax.length / (2.0 * np.pi)))
    else:
        modes = np.arange(1, n_modes + 1, dtype=float)
    N, E = ax.degree, ax.elements
    xi = torch.as_tensor(np.array(grid.bases[0].nodes[:N]), device=device)
    e = torch.arange(E, dtype=torch.float64, device=device)
    x = (e[:, None] * grid.h + grid.h * (xi[None, :] + 1.0) / 2.0).reshape(-1)
    if not grid.periodic:
        x = torch.cat([x, torch.tensor([E * grid.h], dtype=torch.float64, device=device)])
    out = torch.zeros_like(x)
    for a, m in zip(amps, modes):
        out += float(a) * torch.sin((2.0 * np.pi * float(m) / ax.length) * x)
    return out


def cfg_operator(cfg, device=None, batch=1, bc=PERIODIC):
    grid = grid_1d(cfg["xa"], cfg["xb"], cfg["E"], cfg["N"], bc)
    return SemOperator(grid, PdeCoefficients(cfg["nu"]), device=device, batch=batch)


def cfg4_problem(B=None, steps=None, scheme="rk4", device=None, seed=CFG4["seed"]):
    """BASELINE config 4: B periodic rings (E=256, N=15, nu=0.01) on [0, 20]; u0 and the
    observation IC are sums of 4 seeded Fourier modes (different seeds); observations come
    from a forward run.  ``B``/``steps`` override the sizes for tests."""
    import torch
    c = CFG4
    B = c["B"] if B is None else B
    steps = c["steps"] if steps is None else steps
    grid = grid_1d(c["xa"], c["xb"], c["E"], c["N"], PERIODIC)
    op = SemOperator(grid, PdeCoefficients(c["nu"]), device=device, batch=B)
    ts = timeloop.TsConfig(scheme=scheme, t0=0.0, t_end=steps * c["dt"], dt=c["dt"])
    u0 = fourier_fields(grid, B, 4, seed)
    obs0 = fourier_fields(grid, B, 4, seed + 1000)
    target = timeloop.integrate_ensemble(op, torch.from_numpy(obs0).to(op.device), ts,
                                         store_trajectory=False).u_final
    return AssimilationProblem(name=f"cfg4-{scheme}", grid=grid, op=op, ts=ts, u_target=target,
                               u_guess=u0)


def cfg5_problem(E=None, steps=None, slots=None, device=None, seed=CFG5["seed"], band=None, amp=1.0 / 8.0):
    """BASELINE config 5 (single-GPU form): periodic ring of E elements (h = 1/64, N = 7,
    nu = 1e-3); u0 = 32-mode smooth Fourier field, target = forward run of a perturbed u0.
    ``band``: wavenumber band of the modes (fourier_field_device); ``amp``: scale of u0 (the
    perturbation is amp / 5)."""
    import torch
    c = CFG5
    E = c["E"] if E is None else E
    steps = c["steps"] if steps is None else steps
    slots = c["slots"] if slots is None else slots
    grid = grid_1d(0.0, E * c["h"], E, c["N"], PERIODIC)
    op = SemOperator(grid, PdeCoefficients(c["nu"]), device=device)
    ts = timeloop.TsConfig(scheme="rk4", t0=0.0, t_end=steps * c["dt"], dt=c["dt"])
    u0_t = fourier_field_device(grid, c["modes"], seed, op.device, band) * amp
    pert = fourier_field_device(grid, c["modes"], seed + 77, op.device, band) * (amp / 5.0)
    target = timeloop.integrate(op, u0_t + pert, ts, store_steps=None).u_final
    del pert
    return AssimilationProblem(name="cfg5", grid=grid, op=op, ts=ts, u_target=target,
                               u_guess=u0_t, checkpoint_slots=slots)
