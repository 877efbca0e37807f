"""AssimilationProblem.evaluate on ring-resident problems (config 1's size, batched rings):
forward sweep, terminal seed and backward sweep launched back to back with every check read
in one device->host transfer.  Same values, exceptions and cost counters as the stepwise
path (use_ensemble=False, which checks after every call like the reference)."""

import numpy as np
import pytest

import paper_1806_01422_b200 as sb
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import rel_err

pytestmark = pytest.mark.gpu


def _prob(batch=1, scheme="rk4", dt=1e-4, steps=20, target=None, ensemble=True, bc="periodic"):
    grid = grid_1d(-1.0, 1.0, 16, 9, bc)
    op = sb.SemOperator(grid, sb.PdeCoefficients(0.01), device="cuda:0", batch=batch)
    x = grid.node_coordinates()[0]
    if target is None:
        target = np.stack([np.sin(np.pi * x + 0.3 * b) for b in range(batch)]) if batch > 1 else np.sin(np.pi * x)
    ts = sb.TsConfig(scheme=scheme, t0=0.0, t_end=steps * dt, dt=dt)
    return sb.AssimilationProblem(name="ring", grid=grid, op=op, ts=ts, u_target=_mask(grid, target),
                                  u_guess=None, use_ensemble=ensemble), x


def _mask(grid, a):
    a = np.asarray(a, dtype=float)
    return grid.mask(a) if a.ndim == 1 else np.stack([grid.mask(r) for r in a])


def _u0(x, batch):
    u = np.stack([np.sin(np.pi * x) + 0.1 * np.cos((b + 2) * np.pi * x) for b in range(batch)])
    return u[0] if batch == 1 else u


@pytest.mark.parametrize("batch", [1, 3])
@pytest.mark.parametrize("scheme", ["rk4", "rk3", "euler"])
@pytest.mark.parametrize("bc", ["periodic", "dirichlet0"])
def test_ring_resident_evaluate_matches_stepwise(cuda, batch, scheme, bc):
    pa, x = _prob(batch, scheme, bc=bc)
    pb, _ = _prob(batch, scheme, bc=bc, ensemble=False)
    u0 = _mask(pa.grid, _u0(x, batch))
    ja, ga = pa.evaluate(u0)
    if batch == 1:
        jb, gb = pb.evaluate(u0)
        assert isinstance(ja, float) and isinstance(ga, np.ndarray)
        assert abs(ja - jb) <= 1e-12 * abs(jb) and rel_err(ga, gb) <= 1e-12
        assert pa.op.counters == pb.op.counters
    else:
        import torch
        assert isinstance(ja, torch.Tensor) and ga.shape == u0.shape
        for b in range(batch):       # per problem against a batch-1 stepwise run
            pc, _ = _prob(1, scheme, bc=bc, ensemble=False,
                          target=np.sin(np.pi * x + 0.3 * b))
            jc, gc = pc.evaluate(u0[b])
            assert abs(float(ja[b]) - jc) <= 1e-12 * abs(jc) and rel_err(ga[b], gc) <= 1e-12
    assert pa.last_forward is not None and pa.last_forward.stats["failed"] == []


@pytest.mark.parametrize("batch", [1, 3])
def test_ring_resident_evaluate_failures(cuda, batch):
    import torch
    pa, x = _prob(batch)
    u0 = _u0(x, batch)
    bad = u0.copy()
    bad.reshape(-1)[5] = np.nan
    with pytest.raises(sb.NumericFailure, match="initial state"):
        pa.evaluate(bad)
    assert all(v == 0 for v in pa.op.counters.values())
    # NaN target -> NaN terminal cotangent -> the sweep's cotangent check
    t = pa.u_target.copy()
    t.reshape(-1)[7] = np.nan
    pn, _ = _prob(batch, target=t)
    with pytest.raises(sb.NumericFailure, match="cotangent"):
        pn.evaluate(u0)
    s = 4
    assert pn.op.counters["rhs"] == s * 20 and pn.op.counters["jact"] == 0
    # a blow-up inside the sweep: batches report it, a single ring re-runs stepwise and
    # raises like the reference's integrator
    pf, _ = _prob(batch, dt=0.5, steps=4)
    with pytest.raises((sb.NumericFailure, sb.StepFailure)):
        pf.evaluate(1e150 * u0)
    # a later good evaluate on the same problem works
    j, g = pa.evaluate(u0)
    assert np.all(np.isfinite(np.asarray(g.cpu() if isinstance(g, torch.Tensor) else g)))
