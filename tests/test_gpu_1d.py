"""GPU parity of the 1D path (configs 0 and 1) against the fp64 oracle, through the C ABI.

Tolerances (BASELINE.json north_star): per-operator 1e-5 relative L2 on the
fp32 inner path, 1e-12 on the fp64 outer residual; per-cycle residual
histories within 1e-3 relative until the residual reaches 1e-6; transfer
index maps bit-exact.
"""
import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, history_close, oracle_hierarchy, rel_l2, weights_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_01064_b200 as nmg  # noqa: E402
from oracle import nmg_oracle as O  # noqa: E402

DEV = torch.device("cuda:0")
CFG0 = ni.CONFIGS[0]
CFG1 = ni.CONFIGS[1]


def T(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


@pytest.fixture(scope="module")
def cfg0():
    f = ni.operator_factors(CFG0)
    W = weights_for(CFG0, "seed")
    return f, W, oracle_hierarchy(CFG0, f, W), gpu_hierarchy(CFG0, f, W, max_rhs=256)


@pytest.fixture(scope="module")
def cfg1():
    f = ni.operator_factors(CFG1)
    W = weights_for(CFG1, "seed")
    return f, W, oracle_hierarchy(CFG1, f, W), gpu_hierarchy(CFG1, f, W, max_rhs=CFG1.nrhs)


# ------------------------------------------------------------------ transfers: bit-exact
@pytest.mark.parametrize("nrhs", [1, 5])
def test_transfers_bit_exact(cfg0, nrhs):
    _, _, H, h = cfg0
    rng = np.random.default_rng(0)
    for lvl in range(1, CFG0.levels):
        n = CFG0.n >> (lvl - 1)
        f = rng.integers(-64, 64, size=(nrhs, n)).astype(np.float32)   # exact in fp32 sums
        out = torch.zeros(nrhs, n // 2, device=DEV)
        h.debug_op(lvl, nmg.OP_RESTRICT, T(f), out)
        want = O.restrict(H, lvl - 1, f.astype(np.float64))
        assert np.array_equal(out.cpu().numpy().astype(np.float64), want)
        c = rng.integers(-64, 64, size=(nrhs, n // 2)).astype(np.float32)
        base = rng.integers(-64, 64, size=(nrhs, n)).astype(np.float32)
        acc = T(base)
        h.debug_op(lvl, nmg.OP_PROLONG, T(c), acc)
        want = base.astype(np.float64) + O.interpolate(H, lvl - 1, c.astype(np.float64))
        assert np.array_equal(acc.cpu().numpy().astype(np.float64), want)


def test_transfer_index_maps_unit_vectors(cfg0):
    """Index maps and weights: the GPU restriction/prolongation of unit vectors
    reproduce the oracle's R and P matrices entry for entry."""
    _, _, H, h = cfg0
    n = CFG0.n
    E = np.eye(n, dtype=np.float32)
    out = torch.zeros(n, n // 2, device=DEV)
    h.debug_op(1, nmg.OP_RESTRICT, T(E), out)
    assert np.array_equal(out.cpu().numpy().T.astype(np.float64), H.R[0])
    Ec = np.eye(n // 2, dtype=np.float32)
    acc = torch.zeros(n // 2, n, device=DEV)
    h.debug_op(1, nmg.OP_PROLONG, T(Ec), acc)
    assert np.array_equal(acc.cpu().numpy().T.astype(np.float64), H.P[0])


# ------------------------------------------------------------------ per-operator parity
@pytest.mark.parametrize("nrhs", [1, 7, 130])
def test_apply_and_residual(cfg0, nrhs):
    _, _, H, h = cfg0
    rng = np.random.default_rng(1)
    for lvl in range(1, CFG0.levels):
        n = CFG0.n >> (lvl - 1)
        x = rng.standard_normal((nrhs, n)).astype(np.float32)
        out = torch.zeros(nrhs, n, device=DEV)
        h.debug_op(lvl, nmg.OP_APPLY, T(x), out)
        want = O.apply_A(H, lvl - 1, x.astype(np.float64))
        assert rel_l2(out.cpu().numpy(), want) < 1e-5
        y = rng.standard_normal((nrhs, n)).astype(np.float32)
        r = T(y)
        h.debug_op(lvl, nmg.OP_RESIDUAL, T(x), r)
        assert rel_l2(r.cpu().numpy(), y - want) < 1e-5


@pytest.mark.parametrize("lvl", [1, 2, 3, 4, 5])
def test_apply_cfg1_levels_ragged(cfg1, lvl):
    """tcgen05 3xTF32 operator apply at every smoothed level of config 1, ragged batch."""
    _, _, H, h = cfg1
    n = CFG1.n >> (lvl - 1)
    nrhs = 131
    rng = np.random.default_rng(10 + lvl)
    x = rng.standard_normal((nrhs, n)).astype(np.float32)
    y = rng.standard_normal((nrhs, n)).astype(np.float32)
    want = O.apply_A(H, lvl - 1, x.astype(np.float64))
    out = torch.zeros(nrhs, n, device=DEV)
    h.debug_op(lvl, nmg.OP_APPLY, T(x), out)
    assert rel_l2(out.cpu().numpy(), want) < 1e-5
    r = T(y)
    h.debug_op(lvl, nmg.OP_RESIDUAL, T(x), r)
    assert rel_l2(r.cpu().numpy(), y - want) < 1e-5


def test_filter(cfg0):
    _, _, H, h = cfg0
    rng = np.random.default_rng(2)
    for lvl in range(1, CFG0.levels):
        n = CFG0.n >> (lvl - 1)
        x = rng.standard_normal((6, n)).astype(np.float32)
        out = torch.zeros(6, n, device=DEV)
        h.debug_op(lvl, nmg.OP_FILTER, T(x), out)
        assert rel_l2(out.cpu().numpy(), O.level_filter(H, lvl - 1, x.astype(np.float64))) < 2e-6


@pytest.mark.parametrize("n", [256, 4096])
def test_cnn_and_smooth(cfg0, cfg1, n):
    cfg, (f, W, H, h) = (CFG0, cfg0) if n == 256 else (CFG1, cfg1)
    rng = np.random.default_rng(3)
    nrhs = 9
    u = rng.standard_normal((nrhs, n)).astype(np.float32)
    out = torch.zeros(nrhs, n, device=DEV)
    h.debug_op(1, nmg.OP_CNN, T(u), out)
    want = O.cnn_forward(H.weights[0], u.astype(np.float64))
    assert rel_l2(out.cpu().numpy(), want) < 1e-5
    b = (3.7 * rng.standard_normal((nrhs, n))).astype(np.float32)
    x0 = rng.standard_normal((nrhs, n)).astype(np.float32)
    xs = T(x0)
    h.debug_op(1, nmg.OP_SMOOTH, T(b), xs)
    s = np.linalg.norm(b.astype(np.float64), axis=1, keepdims=True)
    hv = O.cnn_forward(H.weights[0], b / s) * s
    want = x0 + O.level_filter(H, 0, hv)
    assert rel_l2(xs.cpu().numpy() - x0, want - x0) < 1e-5


def test_smooth_zero_rhs_guard(cfg0):
    _, _, _, h = cfg0
    x = torch.ones(3, CFG0.n, device=DEV)
    h.debug_op(1, nmg.OP_SMOOTH, torch.zeros(3, CFG0.n, device=DEV), x)
    assert torch.equal(x, torch.ones_like(x))


def test_coarse_solve(cfg0):
    _, _, H, h = cfg0
    nc = CFG0.n >> (CFG0.levels - 1)
    y = np.random.default_rng(4).standard_normal((11, nc)).astype(np.float32)
    out = torch.zeros(11, nc, device=DEV)
    h.debug_op(CFG0.levels, nmg.OP_COARSE, T(y), out)
    assert rel_l2(out.cpu().numpy(), O.coarse_solve(H, y.astype(np.float64))) < 1e-6


@pytest.mark.parametrize("nrhs", [5, 72])
def test_outer_residual_fp64(cfg0, cfg1, nrhs):
    """fp64 outer residual within 1e-12: DMMA for small batches (nrhs <= 64), exact int8 digit
    products on tcgen05 (Ozaki) above."""
    for cfg, (f, W, H, h) in ((CFG0, cfg0), (CFG1, cfg1)):
        rng = np.random.default_rng(5)
        y = rng.standard_normal((nrhs, cfg.n))
        x = rng.standard_normal((nrhs, cfg.n))
        r = torch.zeros(nrhs, cfg.n, dtype=torch.float64, device=DEV)
        rr = torch.zeros(nrhs, dtype=torch.float64, device=DEV)
        h.residual(T(y, torch.float64), T(x, torch.float64), r, rr)
        want = y - O.apply_A(H, 0, x)
        assert rel_l2(r.cpu().numpy(), want) < 1e-12
        assert np.allclose(rr.cpu().numpy(), np.linalg.norm(want, axis=1) / np.linalg.norm(y, axis=1), rtol=1e-12)


def test_outer_residual_wide_dynamic_range(cfg1):
    """The fp64 residual is emulated with exact int8 digit products (7 digits per operand,
    per-row exponents): entries spanning 11 decades in one row still give a residual within
    1e-12 of the fp64 oracle, relative to ||y|| + ||A|| ||x||."""
    f, W, H, h = cfg1
    rng = np.random.default_rng(6)
    nrhs = 72                                   # > 64: the Ozaki path
    x = rng.standard_normal((nrhs, CFG1.n)) * 10.0 ** rng.uniform(-8, 3, size=(nrhs, CFG1.n))
    y = O.apply_A(H, 0, x) + 1e-6 * rng.standard_normal((nrhs, CFG1.n))   # near-converged
    r = torch.zeros(nrhs, CFG1.n, dtype=torch.float64, device=DEV)
    h.residual(T(y, torch.float64), T(x, torch.float64), r, None)
    want = y - O.apply_A(H, 0, x)
    scale = np.linalg.norm(y, axis=1) + np.abs(H.A[0]).sum(1).max() * np.abs(x).max(axis=1)
    err = np.linalg.norm(r.cpu().numpy() - want, axis=1) / scale
    assert err.max() < 1e-12, err


def test_inner_cycle_from_zero(cfg0):
    """NMGF(0, y) in fp32 vs the oracle's fp64 cycle (whole inner V-cycle)."""
    f, W, H, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    out = torch.zeros(y.shape, device=DEV)
    h.debug_op(1, nmg.OP_CYCLE0, T(y.astype(np.float32)), out)
    want = O.nmgf_cycle(H, np.zeros_like(y), y.astype(np.float32).astype(np.float64))
    assert rel_l2(out.cpu().numpy(), want) < 1e-4


# ------------------------------------------------------------------ residual histories
def _gpu_solve(h, y, max_cycles, tol=1e-300):
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=tol, max_cycles=max_cycles)
    return rep, xd.cpu().numpy()


def test_cfg0_wseed_history(cfg0):
    f, W, H, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    rep, x = _gpu_solve(h, y, CFG0.cycles)
    orc = O.solve(H, y, tol=1e-300, max_cycles=CFG0.cycles, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err
    assert rel_l2(x, orc.x) < 1e-3


def test_cfg0_wlin_solve_matches():
    f = ni.operator_factors(CFG0)
    W = weights_for(CFG0, "lin")
    H = oracle_hierarchy(CFG0, f, W)
    h = gpu_hierarchy(CFG0, f, W, max_rhs=8)
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    orc = O.solve(H, y, tol=1e-6, max_cycles=80)
    rep, x = _gpu_solve(h, y, 80, tol=1e-6)
    assert rep["converged"].all() and orc.converged.all()
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err
    d = np.abs(rep["cycles"] - orc.cycles)
    # same stopping cycle; +-1 only when the oracle residual sits within 1e-3 of tol
    for b in np.nonzero(d)[0]:
        assert d[b] == 1
        c = min(rep["cycles"][b], orc.cycles[b])
        assert abs(orc.history[b, c] - 1e-6) <= 1e-3 * 1e-6 * 10


@pytest.mark.parametrize("alpha", ni.ALPHAS[1])
def test_cfg1_wseed_history_subset(alpha):
    cfg = CFG1.replace(alpha=alpha)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=4)
    y, _ = ni.make_rhs(cfg, f, alpha, nrhs=4)
    rep, _ = _gpu_solve(h, y, cfg.cycles)
    orc = O.solve(H, y, tol=1e-300, max_cycles=cfg.cycles, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_cfg1_full_batch_sampled(cfg1):
    """Full BASELINE size (1024 RHS, the bench launch configuration): one cycle on
    the GPU, sampled RHS checked against the oracle run on those RHS alone."""
    f, W, H, h = cfg1
    y, _ = ni.make_rhs(CFG1, f, CFG1.alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    h.vcycle(yd, xd)
    h.vcycle(yd, xd)
    idx = [0, 1, 511, 1023]
    orc = O.nmgf_cycle(H, np.zeros((4, CFG1.n)), y[idx])
    orc = O.nmgf_cycle(H, orc, y[idx])
    got = xd.cpu().numpy()[idx]
    assert rel_l2(got, orc) < 1e-3
    rg = O.relative_residual(H, got, y[idx])
    ro = O.relative_residual(H, orc, y[idx])
    assert np.all(np.abs(rg - ro) <= 1e-3 * ro)


# ------------------------------------------------------------------ metamorphic / edge cases
def test_homogeneity_bitwise(cfg0):
    f, W, H, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    outs = []
    for s in (1.0, 8.0, 2.0 ** -5):
        yd = T(s * y, torch.float64)
        xd = torch.zeros_like(yd)
        h.vcycle(yd, xd)
        h.vcycle(yd, xd)
        outs.append(xd.cpu().numpy() / s)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_batch_invariance_bitwise(cfg0):
    f, W, H, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    yb = np.concatenate([y] * 5)[:37]                 # ragged batch
    yd = T(yb, torch.float64)
    xd = torch.zeros_like(yd)
    h.vcycle(yd, xd)
    for i in (0, 3, 36):
        y1 = T(yb[i:i + 1], torch.float64)
        x1 = torch.zeros_like(y1)
        h.vcycle(y1, x1)
        assert torch.equal(x1[0], xd[i])


def test_zero_rhs_and_empty_batch(cfg0):
    _, _, _, h = cfg0
    yd = torch.zeros(3, CFG0.n, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, max_cycles=3)
    assert rep["converged"].all() and torch.count_nonzero(xd) == 0
    e = torch.zeros(0, CFG0.n, dtype=torch.float64, device=DEV)
    h.vcycle(e, e.clone())


def test_nan_reported_for_its_rhs(cfg0):
    f, _, _, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    y[5, 17] = np.nan
    yd = T(y, torch.float64)
    with pytest.raises(nmg.NmgError) as ei:
        h.solve(yd, torch.zeros_like(yd), max_cycles=3)
    assert ei.value.status == 5 and ei.value.report["fail_rhs"] == 5


def test_host_entry_matches_device(cfg0):
    f, _, _, h = cfg0
    y, _ = ni.make_rhs(CFG0, f, CFG0.alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    for _ in range(3):
        h.vcycle(yd, xd)
    xh = np.zeros_like(y)
    h.vcycles_host(np.ascontiguousarray(y), xh, 3)
    assert np.array_equal(xh, xd.cpu().numpy())


def test_host_entry_chunked_pipeline():
    """nmg_vcycles_host splits >= 256 RHS into chunks whose copies overlap the cycles of the
    previous chunk; per-RHS independence makes the result bitwise equal to one device call."""
    cfg = CFG0.replace(nrhs=600)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    h = gpu_hierarchy(cfg, f, W, max_rhs=600)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    for _ in range(2):
        h.vcycle(yd, xd)
    xh = np.zeros_like(y)
    h.vcycles_host(np.ascontiguousarray(y), xh, 2)
    assert np.array_equal(xh, xd.cpu().numpy())


@pytest.mark.parametrize("host_chunks", [0, 2])
def test_host_entry_lanes(host_chunks):
    """On a handle with RHS lanes (max_rhs 1024: four lanes of 256) nmg_vcycles_host either
    pipelines the copies per lane (default: a lane cycles as soon as its RHS land) or per chunk
    (tuning.host_chunks, lanes inside each chunk); x is bitwise the device-entry result and relres
    (the relative residual before the last cycle, every lane's slice) matches nmg_residual."""
    cfg = ni.CONFIGS[1].replace(n=1024, levels=4, nrhs=1024)
    f = ni.operator_factors(cfg)
    W = ni.weights_seed(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=1024)
    h = nmg.Hierarchy(1, cfg.n, cfg.levels, cfg.alpha, f, nu1=1, nu2=1, max_rhs=1024,
                      tuning={"host_chunks": host_chunks})
    for l, w in enumerate(W):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    st = torch.cuda.Stream()
    h.vcycle(yd, xd, st)
    h.vcycle(yd, xd, st)
    rr_ref = torch.empty(1024, dtype=torch.float64, device=DEV)
    h.residual(yd, xd, relres=rr_ref, stream=st)
    h.vcycle(yd, xd, st)
    torch.cuda.synchronize()
    xh = np.zeros_like(y)
    rr = np.zeros(1024)
    h.vcycles_host(np.ascontiguousarray(y), xh, 3, relres=rr, stream=st)
    assert np.array_equal(xh, xd.cpu().numpy())
    np.testing.assert_allclose(rr, rr_ref.cpu().numpy(), rtol=1e-12, atol=0)
    h.close()


def test_rhs_lanes_bitwise():
    """Batches >= 256 RHS on a handle with max_rhs >= 512 run as two RHS lanes on forked
    streams (nmg_vcycle); the NMGF cycle is per-RHS, so the result is bitwise the one-lane result."""
    cfg = ni.CONFIGS[1].replace(n=1024, levels=4, nrhs=512)
    f = ni.operator_factors(cfg)
    W = ni.weights_seed(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=512)
    outs = []
    for lanes in (1, 0):
        h = nmg.Hierarchy(1, cfg.n, cfg.levels, cfg.alpha, f, nu1=1, nu2=1, max_rhs=512,
                          tuning={"lanes": lanes})
        for l, w in enumerate(W):
            h.load_weights(l + 1, ni.cnn_arch(cfg), w)
        yd = torch.tensor(y, dtype=torch.float64, device=DEV)
        xd = torch.zeros_like(yd)
        st = torch.cuda.Stream()
        for _ in range(3):                     # eager, capture, replay
            h.vcycle(yd, xd, st)
        torch.cuda.synchronize()
        outs.append(xd.cpu().numpy())
        h.close()
    assert np.array_equal(outs[0], outs[1])
