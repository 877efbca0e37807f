"""Operator parity on the B200: F, J v, J^T w through the C ABI vs the reference
fixtures and the oracle.  Tolerances (BASELINE north_star): 1e-12 relative (max-abs,
normalised by the reference's max) per apply on the BASELINE's rough inputs;
integer maps and the gather bit-exact."""

import numpy as np
import pytest
import torch

import paper_1806_01422_b200 as sb
from oracle import semref as R
from paper_1806_01422_b200 import configs
from paper_1806_01422_b200.grid import grid_1d
from semtest_util import golden, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _op(xa, xb, E, N, periodic, nu, batch=1):
    g = grid_1d(xa, xb, int(E), int(N), "periodic" if periodic else "dirichlet0")
    return sb.SemOperator(g, sb.PdeCoefficients(nu), device="cuda:0", batch=batch)


def test_golden_operator_cases(cuda):
    g = golden("ops.npz")
    k = 0
    while f"case_{k}" in g:
        xa, xb, E, N, per, nu, _ = g[f"case_{k}"]
        op = _op(xa, xb, E, N, per, nu)
        u, v, w = g[f"u_{k}"], g[f"v_{k}"], g[f"w_{k}"]
        assert rel_err(op.apply_rhs(u), g[f"f_{k}"]) <= TOL, k
        assert rel_err(op.apply_jacobian(u, v), g[f"jv_{k}"]) <= TOL, k
        assert rel_err(op.apply_jacobian_transpose(u, w), g[f"jtw_{k}"]) <= TOL, k
        assert op.counters == {"rhs": 1, "jac": 1, "jact": 1}
        k += 1


@pytest.mark.parametrize("N", list(range(1, 33)))
@pytest.mark.parametrize("periodic", [True, False])
def test_every_degree_vs_oracle(cuda, N, periodic):
    # element counts straddle the CTA tile (256 / 128 elements) to exercise halos and tails
    E = {1: 700, 2: 300}.get(N, 261 if N <= 8 else 131)
    nu = 0.01
    op = _op(-1.0, 1.0, E, N, periodic, nu)
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, periodic), nu)
    u, v, w = R.seeded_fields(ref.mesh.ndof, 100 + N)
    assert rel_err(op.apply_rhs(u), ref.rhs(u)) <= TOL
    assert rel_err(op.apply_jacobian(u, v), ref.jac(u, v)) <= TOL
    assert rel_err(op.apply_jacobian_transpose(u, w), ref.jact(u, w)) <= TOL


@pytest.fixture(params=[0, 1, 2, 3], ids=["auto", "no-mma", "plain", "mma-sync"])
def kernel_path(request):
    from paper_1806_01422_b200 import _lib
    lib = _lib.load()
    assert lib.sem1d_set_kernel_path(request.param) == 0
    yield request.param
    lib.sem1d_set_kernel_path(0)


@pytest.mark.parametrize("N", [1, 3, 5, 7, 9, 11, 15, 21, 23, 31])
@pytest.mark.parametrize("periodic", [True, False])
def test_tma_pipeline_vs_oracle(cuda, N, periodic, kernel_path):
    """Large rings take the persistent pipelined kernels (DMMA tensor-core path for
    N+1 in {8, 16, 24, 32}, TMA/DFMA path for other odd N); every path is checked:
    ragged tails, batch > 1 and both boundary kinds."""
    tpb = 256 if N <= 8 else 128
    E = 7 * tpb + 37
    B = 3
    op = _op(-1.0, 1.0, E, N, periodic, 0.01, batch=B)
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, E, N, periodic), 0.01)
    rng = np.random.default_rng(N)
    U = rng.uniform(-1, 1, (B, ref.mesh.ndof))
    V = rng.standard_normal((B, ref.mesh.ndof))
    W = rng.standard_normal((B, ref.mesh.ndof))
    F, JV, JT = op.apply_rhs(U), op.apply_jacobian(U, V), op.apply_jacobian_transpose(U, W)
    for b in range(B):
        assert rel_err(F[b], ref.rhs(U[b])) <= TOL
        assert rel_err(JV[b], ref.jac(U[b], V[b])) <= TOL
        assert rel_err(JT[b], ref.jact(U[b], W[b])) <= TOL
    bad = U.copy()
    bad[1, ref.mesh.ndof // 2] = np.nan
    with pytest.raises(sb.NumericFailure):
        op.apply_rhs(bad)


@pytest.mark.parametrize("E", [1, 2, 3, 255, 256, 257, 512, 1000])
def test_tile_edges(cuda, E):
    for periodic in (True, False):
        N = 7 if (periodic or E > 0) else 7
        if periodic and E * N < 2:
            continue
        op = _op(0.0, 3.0, E, N, periodic, 0.02)
        ref = R.BurgersOracle(R.Mesh1D(0.0, 3.0, E, N, periodic), 0.02)
        u, v, w = R.seeded_fields(ref.mesh.ndof, E)
        assert rel_err(op.apply_rhs(u), ref.rhs(u)) <= TOL
        assert rel_err(op.apply_jacobian(u, v), ref.jac(u, v)) <= TOL
        assert rel_err(op.apply_jacobian_transpose(u, w), ref.jact(u, w)) <= TOL


@pytest.mark.parametrize("N", [15, 31])
@pytest.mark.parametrize("E", [1, 2, 3, 5, 17])
def test_tiny_rings_on_the_split_kernels(cuda, N, E):
    """N = 15 / 31 take the reflection-split DMMA kernel at every ring size: rings smaller than
    one m-tile, wrap-around of a one- or two-element periodic ring, both boundary kinds,
    batches (rows 0 and N of an element sit in the same lane there)."""
    for periodic in (True, False):
        for B in (1, 3):
            op = _op(0.0, 3.0, E, N, periodic, 0.02, batch=B)
            ref = R.BurgersOracle(R.Mesh1D(0.0, 3.0, E, N, periodic), 0.02)
            rng = np.random.default_rng(100 * N + E)
            U = rng.uniform(-1, 1, (B, ref.mesh.ndof))
            V = rng.standard_normal((B, ref.mesh.ndof))
            F = op.apply_rhs(U if B > 1 else U[0])
            JV = op.apply_jacobian(U if B > 1 else U[0], V if B > 1 else V[0])
            JT = op.apply_jacobian_transpose(U if B > 1 else U[0], V if B > 1 else V[0])
            for b in range(B):
                f, jv, jt = (x[b] if B > 1 else x for x in (F, JV, JT))
                assert rel_err(f, ref.rhs(U[b])) <= TOL
                assert rel_err(jv, ref.jac(U[b], V[b])) <= TOL
                assert rel_err(jt, ref.jact(U[b], V[b])) <= TOL


def test_batched_operator_equals_per_problem(cuda):
    B, E, N = 5, 40, 15
    op = _op(0.0, 20.0, E, N, True, 0.01, batch=B)
    ref = R.BurgersOracle(R.Mesh1D(0.0, 20.0, E, N, True), 0.01)
    rng = np.random.default_rng(5)
    U = rng.uniform(-1, 1, (B, ref.mesh.ndof))
    W = rng.standard_normal((B, ref.mesh.ndof))
    F = op.apply_rhs(U)
    JT = op.apply_jacobian_transpose(U, W)
    for b in range(B):
        assert rel_err(F[b], ref.rhs(U[b])) <= TOL
        assert rel_err(JT[b], ref.jact(U[b], W[b])) <= TOL


def test_scatter_gather_bit_exact(cuda):
    for per in (True, False):
        for E, N in [(1, 3), (2, 1), (16, 9), (300, 7)]:
            if per and E * N < 2:
                continue
            grid = grid_1d(-1.0, 1.0, E, N, "periodic" if per else "dirichlet0")
            m = R.Mesh1D(-1.0, 1.0, E, N, per)
            rng = np.random.default_rng(E * 31 + N)
            u = rng.standard_normal(grid.nglobal)
            loc = rng.standard_normal((1, E, N + 1))
            assert np.array_equal(grid.scatter(u)[0], m.localize(u))
            assert np.array_equal(grid.gather(loc), m.assemble(loc[0]))
            ones = np.ones((1, E, N + 1))
            assert np.array_equal(grid.gather(ones), grid.multiplicity)


def test_nonfinite_inputs_raise(cuda):
    op = _op(-1.0, 1.0, 16, 9, True, 0.01)
    u = np.zeros(op.ndof)
    bad = u.copy()
    bad[77] = np.nan
    with pytest.raises(sb.NumericFailure, match="state"):
        op.apply_rhs(bad)
    with pytest.raises(sb.NumericFailure, match="tangent"):
        op.apply_jacobian(u, bad)
    bad[77] = np.inf
    with pytest.raises(sb.NumericFailure, match="cotangent"):
        op.apply_jacobian_transpose(u, bad)
    op.apply_rhs(u)  # flag was cleared
    with pytest.raises(sb.ValidationError):
        op.apply_rhs(np.zeros(op.ndof + 1))


def test_operator_properties(cuda):
    """SPEC.md ops invariants: F(const) = 0, 1^T M f = 0 (periodic), J linear in w,
    J vs central FD, dot-product identity, densify^T z = J^T z."""
    op = _op(-1.0, 1.0, 3, 4, True, 0.01)
    n = op.ndof
    assert np.max(np.abs(op.apply_rhs(np.full(n, 0.7)))) <= 1e-13
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, n)
    f = op.apply_rhs(u)
    assert abs(op.grid.mass_scalar @ f) <= 1e-12 * np.abs(op.grid.mass_scalar * f).sum()
    w = rng.standard_normal(n)
    eps = 1e-5
    fd = (op.apply_rhs(u + eps * w) - op.apply_rhs(u - eps * w)) / (2 * eps)
    assert rel_err(fd, op.apply_jacobian(u, w)) <= 1e-8
    for per in (True, False):
        op = _op(-1.0, 1.0, 3, 4, per, 0.01)
        mask = op.grid.mask_scalar
        for _ in range(200):
            u, w, z = (rng.standard_normal(op.ndof) * mask for _ in range(3))
            lhs = op.apply_jacobian(u, w) @ z
            rhs = w @ op.apply_jacobian_transpose(u, z)
            assert abs(lhs - rhs) / (np.linalg.norm(w) * np.linalg.norm(z)) <= 1e-13
        Jd = op.densify(u)
        # J^T output is masked at Dirichlet ends (ops.py:257): compare on the mask
        assert rel_err(mask * (Jd.T @ z), op.apply_jacobian_transpose(u, z)) <= 1e-12


def test_device_tensors_in_device_tensors_out(cuda):
    op = _op(-1.0, 1.0, 64, 7, True, 0.01)
    u = torch.rand(op.ndof, dtype=torch.float64, device=cuda)
    f = op.apply_rhs(u)
    assert isinstance(f, torch.Tensor) and f.is_cuda
    assert torch.equal(f, op.apply_rhs(u))  # bitwise reproducible


def test_cfg2_full_size_properties(cuda):
    """BASELINE config 2 at full size (E = 2^22, N = 7): size-independent checks --
    linearity of J and J^T, the dot-product identity, and oracle parity on a
    periodic sub-window computed on the host."""
    c = configs.CFG2
    op = configs.cfg_operator(c, device="cuda:0")
    u, v, w = configs.operator_inputs(op.ndof, c["seed"])
    ud, vd, wd = (torch.from_numpy(a).to(cuda) for a in (u, v, w))
    f = op.apply_rhs(ud)
    jv = op.apply_jacobian(ud, vd)
    jtw = op.apply_jacobian_transpose(ud, wd)
    assert torch.isfinite(f).all() and torch.isfinite(jv).all() and torch.isfinite(jtw).all()
    # linearity
    jv2 = op.apply_jacobian(ud, 2.0 * vd + wd)
    lin = 2.0 * jv + op.apply_jacobian(ud, wd)
    assert float((jv2 - lin).abs().max() / lin.abs().max()) <= 1e-12
    # dot-product identity at full size
    lhs = float(torch.dot(jv, wd))
    rhs = float(torch.dot(vd, jtw))
    # ||J|| ~ nu N^4 / h^2 ~ 1e13 here: normalise by the inner product itself
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # oracle on windows of elements: element-local results away from the window edge
    N, E = c["N"], c["E"]
    fh, jh = f.cpu().numpy(), jtw.cpu().numpy()
    h = (c["xb"] - c["xa"]) / E
    for e0 in (0, E // 2 - 17, E - 64):
        ne = 64
        sub = R.BurgersOracle(R.Mesh1D(0.0, ne * h, ne, N, True), c["nu"])
        idx = (np.arange(e0 * N, (e0 + ne) * N)) % op.ndof
        fs = sub.rhs(u[idx])
        js = sub.jact(u[idx], w[idx])
        inner = slice(N + 1, (ne - 1) * N)   # interior nodes do not see the window wrap
        assert rel_err(fh[idx][inner], fs[inner]) <= TOL
        assert rel_err(jh[idx][inner], js[inner]) <= TOL


@pytest.mark.parametrize("E,N,bc", [(4096, 7, "periodic"), (1000, 15, "dirichlet0"), (600, 9, "periodic")])
def test_host_streaming_apply(cuda, E, N, bc):
    """apply_host: chunked H2D / compute / D2H overlap == device applies (same kernels)."""
    op = _op(-1.0, 1.0, E, N, bc == "periodic", 0.01)
    u, v, w = R.seeded_fields(op.ndof, E)
    uh, vh, wh = (torch.from_numpy(a).pin_memory() for a in (u, v, w))
    out = op.apply_host(uh, vh, wh)
    ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
    for k, ref in (("rhs", op.apply_rhs(ud)), ("jac", op.apply_jacobian(ud, vd)),
                   ("jact", op.apply_jacobian_transpose(ud, wd))):
        assert rel_err(out[k].numpy(), ref.cpu().numpy()) <= 1e-14
    npout = op.apply_host(u, kinds=["rhs"])
    assert np.array_equal(npout["rhs"], out["rhs"].numpy())
    for slots in (2, 4):       # caller-provided outputs, other buffer-set counts
        given = {k: torch.full((op.ndof,), 7.0, dtype=torch.float64).pin_memory() for k in out}
        r = op.apply_host(uh, vh, wh, out=given, slots=slots, chunks=5)
        for k in out:
            assert r[k] is given[k] and torch.equal(given[k], out[k])
    bad = u.copy()
    bad[E] = np.nan
    with pytest.raises(sb.NumericFailure):
        op.apply_host(bad)


def test_max_size_config5_apply(cuda):
    """Largest BASELINE field (config 5: E = 2^25, N = 7, 235M DOF, 1.9 GB per field):
    size-independent properties on device-generated inputs plus oracle windows."""
    from paper_1806_01422_b200 import configs
    c = configs.CFG5
    g = grid_1d(0.0, c["E"] * c["h"], c["E"], c["N"])
    op = sb.SemOperator(g, sb.PdeCoefficients(c["nu"]), device="cuda:0")
    gen = torch.Generator(device="cuda").manual_seed(55)
    u = torch.rand(op.ndof, dtype=torch.float64, device=cuda, generator=gen) * 2 - 1
    v = torch.randn(op.ndof, dtype=torch.float64, device=cuda, generator=gen)
    f = op.apply_rhs(u)
    jv = op.apply_jacobian(u, v)
    jtv = op.apply_jacobian_transpose(u, v)
    assert bool(torch.isfinite(f).all() and torch.isfinite(jv).all() and torch.isfinite(jtv).all())
    # dot-product identity <J v, v> = <v, J^T v> at 235M DOF
    lhs, rhs = float(torch.dot(jv, v)), float(torch.dot(v, jtv))
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)
    # periodic conservation 1^T M f = 0 (SPEC ops invariants), relative to sum |M f|
    m = torch.as_tensor(g.mass_pattern[np.arange(g.axis.degree)], device=cuda).repeat(c["E"])
    mf = m * f
    assert abs(float(mf.sum())) <= 1e-10 * float(mf.abs().sum())
    # oracle windows away from the window edges
    N = c["N"]
    uh, fh = u.cpu().numpy(), f.cpu().numpy()
    for e0 in (0, c["E"] // 3, c["E"] - 64):
        ne = 64
        sub = R.BurgersOracle(R.Mesh1D(0.0, ne * c["h"], ne, N, True), c["nu"])
        idx = np.arange(e0 * N, (e0 + ne) * N) % op.ndof
        inner = slice(N + 1, (ne - 1) * N)
        assert rel_err(fh[idx][inner], sub.rhs(uh[idx])[inner]) <= 1e-12


def test_plan_runs_on_its_own_device(cuda):
    """A plan belongs to the device current at sem1d_plan_create (SemOperator makes its
    `device` current for that); every C-ABI call switches to it and restores the caller's
    device.  On a multi-GPU box the operator is built on the LAST device while device 0 is
    current; on one GPU the guard still must leave the current device untouched."""
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", ndev - 1)
    torch.cuda.set_device(0)
    op = sb.SemOperator(grid_1d(-1.0, 1.0, 700, 7), sb.PdeCoefficients(0.01), device=dev)
    ref = R.BurgersOracle(R.Mesh1D(-1.0, 1.0, 700, 7, True), 0.01)
    u, v, w = R.seeded_fields(ref.mesh.ndof, 9)
    with torch.cuda.device(dev):
        f = op.apply_rhs(u)
        jt = op.apply_jacobian_transpose(u, w)
    assert torch.cuda.current_device() == 0
    assert rel_err(f, ref.rhs(u)) <= TOL and rel_err(jt, ref.jact(u, w)) <= TOL
    ud = torch.from_numpy(u).to(dev)
    out = op.apply_rhs(ud)
    assert out.device == dev and torch.cuda.current_device() == 0


def test_numpy_fields_through_pinned_staging(cuda):
    """Large numpy fields take the pinned-staging path (chunked H2D, pinned result arrays):
    bitwise the same results as device tensors, fresh writable arrays per call, and the
    same validation errors."""
    op = _op(-1.0, 1.0, 1 << 20, 7, True, 0.01)          # 7.3M DOF: 59 MB, several chunks
    u, v, w = R.seeded_fields(op.ndof, 11)
    ud, vd, wd = (torch.from_numpy(a).cuda() for a in (u, v, w))
    for host, dev in ((op.apply_rhs(u), op.apply_rhs(ud)),
                      (op.apply_jacobian(u, v), op.apply_jacobian(ud, vd)),
                      (op.apply_jacobian_transpose(u, w), op.apply_jacobian_transpose(ud, wd))):
        assert isinstance(host, np.ndarray) and host.dtype == np.float64 and host.flags.writeable
        assert np.array_equal(host, dev.cpu().numpy())
    a, b = op.apply_rhs(u), op.apply_rhs(u)
    assert a is not b and not np.shares_memory(a, b)
    a[:] = 0.0
    assert np.array_equal(b, op.apply_rhs(ud).cpu().numpy())
    # a strided / float32 view goes through np.asarray like before
    assert np.array_equal(op.apply_rhs(np.asfortranarray(u.astype(np.float32)).astype(np.float64)),
                          op.apply_rhs(torch.from_numpy(u.astype(np.float32).astype(np.float64)).cuda()).cpu().numpy())
    with pytest.raises(sb.ValidationError):
        op.apply_rhs(u[:-1])


def test_numpy_staging_concurrent_callers(cuda):
    """The pinned staging ring is shared by the process: concurrent drop-in callers
    (ops.py:86-88 allows concurrent calls) still get their own inputs' results."""
    import threading
    op = _op(-1.0, 1.0, 1 << 18, 7, True, 0.01)
    fields = [R.seeded_fields(op.ndof, s)[0] for s in range(4)]
    want = [op.apply_rhs(torch.from_numpy(f).cuda()).cpu().numpy() for f in fields]
    got, errs = [None] * 4, []

    def run(i):
        try:
            for _ in range(3):
                got[i] = op.apply_rhs(fields[i])
        except Exception as e:   # pragma: no cover - surfaced below
            errs.append(e)
    ts = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for i in range(4):
        assert np.array_equal(got[i], want[i]), i
