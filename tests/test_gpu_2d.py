"""GPU parity of the 2D path (configs 2, 3, 4; Alg 4) against the fp64 oracle."""
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
# small 2D cases the oracle finishes in seconds: several tiles, a ragged tile edge (n=48 is
# not a power of two, so use n = 64 with 16x16 CNN tiles and n = 32), B != C (gauss_cos)
SMALL = ni.CONFIGS[2].replace(n=64, levels=3, nrhs=5)
SMALL_COS = ni.CONFIGS[4].replace(n=64, levels=3, nrhs=3, sigma=0.05)


def T(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def _both(cfg, kind="seed", max_rhs=None):
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, kind)
    return f, W, oracle_hierarchy(cfg, f, W), gpu_hierarchy(cfg, f, W, max_rhs=max_rhs or max(cfg.nrhs, 16))


@pytest.fixture(scope="module")
def small():
    return _both(SMALL, max_rhs=64 * 64)


@pytest.fixture(scope="module")
def small_cos():
    return _both(SMALL_COS)


def test_transfers_bit_exact_2d(small):
    _, _, H, h = small
    rng = np.random.default_rng(0)
    for lvl in (1, 2):
        n = SMALL.n >> (lvl - 1)
        f = rng.integers(-64, 64, size=(3, n, n)).astype(np.float32)
        out = torch.zeros(3, n // 2, n // 2, device=DEV)
        h.debug_op(lvl, nmg.OP_RESTRICT, T(f), out)
        assert np.array_equal(out.cpu().numpy().astype(np.float64), O.restrict(H, lvl - 1, f.astype(np.float64)))
        c = rng.integers(-64, 64, size=(3, n // 2, n // 2)).astype(np.float32)
        base = rng.integers(-64, 64, size=(3, n, n)).astype(np.float32)
        acc = T(base)
        h.debug_op(lvl, nmg.OP_PROLONG, T(c), acc)
        want = base + O.interpolate(H, lvl - 1, c.astype(np.float64))
        assert np.array_equal(acc.cpu().numpy().astype(np.float64), want)


@pytest.mark.parametrize("which", ["small", "small_cos"])
def test_apply_2d(which, small, small_cos):
    cfg, (f, W, H, h) = (SMALL, small) if which == "small" else (SMALL_COS, small_cos)
    rng = np.random.default_rng(1)
    for lvl in range(1, cfg.levels):
        n = cfg.n >> (lvl - 1)
        x = rng.standard_normal((3, n, n)).astype(np.float32)
        want = O.apply_A(H, lvl - 1, x.astype(np.float64))
        out = torch.zeros(3, n, n, device=DEV)
        h.debug_op(lvl, nmg.OP_APPLY, T(x), out)
        assert rel_l2(out.cpu().numpy(), want) < 1e-5
        y = rng.standard_normal((3, n, n)).astype(np.float32)
        r = T(y)
        h.debug_op(lvl, nmg.OP_RESIDUAL, T(x), r)
        assert rel_l2(r.cpu().numpy(), y - want) < 1e-5


@pytest.mark.parametrize("n,levels,nrhs", [(128, 4, 3), (512, 6, 2)])
def test_kron_apply_levels(n, levels, nrhs):
    """kron_tc (the 2D Kronecker apply on tcgen05) at every level it serves: mass stencil
    half-bandwidths 0, 1, 2 (Q_0 = I, Q_l = R Q_{l-1} P), ragged 128-row tiles (M = nrhs n),
    and n = 512 (two 256-wide N tiles per row block).  Element-wise against the oracle's
    A_l X = C X B^T + alpha Q X Q^T."""
    cfg = ni.CONFIGS[2].replace(n=n, levels=levels, nrhs=nrhs)
    f, W, H, h = _both(cfg, max_rhs=nrhs)
    rng = np.random.default_rng(7)
    for lvl in range(1, levels):
        m = n >> (lvl - 1)
        x = rng.standard_normal((nrhs, m, m)).astype(np.float32)
        want = O.apply_A(H, lvl - 1, x.astype(np.float64))
        out = torch.zeros(nrhs, m, m, device=DEV)
        h.debug_op(lvl, nmg.OP_APPLY, T(x), out)
        got = out.cpu().numpy().astype(np.float64)
        scale = np.abs(want).max()
        assert np.abs(got - want).max() <= 1e-5 * scale, (lvl, np.abs(got - want).max() / scale)
        y = rng.standard_normal((nrhs, m, m)).astype(np.float32)
        r = T(y)
        h.debug_op(lvl, nmg.OP_RESIDUAL, T(x), r)
        assert np.abs(r.cpu().numpy() - (y - want)).max() <= 1e-5 * max(scale, 1.0), lvl


def test_filter_2d(small):
    _, _, H, h = small
    rng = np.random.default_rng(2)
    for lvl in (1, 2):
        n = SMALL.n >> (lvl - 1)
        x = rng.standard_normal((4, n, n)).astype(np.float32)
        out = torch.zeros(4, n, n, device=DEV)
        h.debug_op(lvl, nmg.OP_FILTER, T(x), out)
        assert rel_l2(out.cpu().numpy(), O.level_filter(H, lvl - 1, x.astype(np.float64))) < 2e-6


def test_cnn_and_smooth_2d(small):
    _, _, H, h = small
    rng = np.random.default_rng(3)
    n = SMALL.n
    u = rng.standard_normal((3, n, n)).astype(np.float32)
    out = torch.zeros(3, n, n, device=DEV)
    h.debug_op(1, nmg.OP_CNN, T(u), out)
    assert rel_l2(out.cpu().numpy(), O.cnn_forward(H.weights[0], u.astype(np.float64))) < 1e-5
    b = (2.5 * rng.standard_normal((3, n, n))).astype(np.float32)
    x0 = rng.standard_normal((3, n, n)).astype(np.float32)
    xs = T(x0)
    h.debug_op(1, nmg.OP_SMOOTH, T(b), xs)
    s = np.sqrt((b.astype(np.float64) ** 2).sum(axis=(1, 2)))[:, None, None]
    hv = O.cnn_forward(H.weights[0], b / s) * s
    want = x0 + O.level_filter(H, 0, hv)
    assert rel_l2(xs.cpu().numpy() - x0, want - x0) < 1e-5


def test_coarse_2d(small):
    _, _, H, h = small
    nc = SMALL.n >> (SMALL.levels - 1)
    y = np.random.default_rng(4).standard_normal((6, nc, nc)).astype(np.float32)
    out = torch.zeros(6, nc, nc, device=DEV)
    h.debug_op(SMALL.levels, nmg.OP_COARSE, T(y), out)
    assert rel_l2(out.cpu().numpy(), O.coarse_solve(H, y.astype(np.float64))) < 1e-6


@pytest.mark.parametrize("which", ["small", "small_cos"])
def test_outer_residual_2d(which, small, small_cos):
    cfg, (f, W, H, h) = (SMALL, small) if which == "small" else (SMALL_COS, small_cos)
    rng = np.random.default_rng(5)
    y = rng.standard_normal((3, cfg.n, cfg.n))
    x = rng.standard_normal((3, cfg.n, cfg.n))
    r = torch.zeros(3, cfg.n, cfg.n, dtype=torch.float64, device=DEV)
    rr = torch.zeros(3, dtype=torch.float64, device=DEV)
    h.residual(T(y, torch.float64), T(x, torch.float64), r, rr)
    want = y - O.apply_A(H, 0, x)
    assert rel_l2(r.cpu().numpy(), want) < 1e-12
    nrm = np.sqrt((want ** 2).sum(axis=(1, 2))) / np.sqrt((y ** 2).sum(axis=(1, 2)))
    assert np.allclose(rr.cpu().numpy(), nrm, rtol=1e-12)


@pytest.mark.parametrize("which", ["small", "small_cos"])
def test_cycle_history_2d_small(which, small, small_cos):
    cfg, (f, W, H, h) = (SMALL, small) if which == "small" else (SMALL_COS, small_cos)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=4)
    orc = O.solve(H, y, tol=1e-300, max_cycles=4, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_homogeneity_and_batch_invariance_2d(small):
    f, _, _, h = small
    y, _ = ni.make_rhs(SMALL, f, SMALL.alpha)
    outs = []
    for s in (1.0, 4.0):
        yd = T(s * y, torch.float64)
        xd = torch.zeros_like(yd)
        h.vcycle(yd, xd)
        outs.append(xd.cpu().numpy() / s)
    assert np.array_equal(outs[0], outs[1])
    # batch invariance (pin P14): every RHS has its own level-filter transform, so a RHS run
    # alone is bitwise its batch result
    for i in (2, 3):
        y1 = T(y[i:i + 1], torch.float64)
        x1 = torch.zeros_like(y1)
        h.vcycle(y1, x1)
        assert np.array_equal(x1.cpu().numpy()[0], outs[0][i])


def test_nan_stays_in_its_rhs_2d(small):
    """A NaN planted in RHS 2 leaves every other RHS of the batch (its level-filter neighbour 3
    included) bitwise unchanged, and nmg_solve reports the failing RHS."""
    f, _, _, h = small
    y, _ = ni.make_rhs(SMALL, f, SMALL.alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    h.vcycle(yd, xd)
    bad = y.copy()
    bad[2, 10, 17] = np.nan
    ybd = T(bad, torch.float64)
    xbd = torch.zeros_like(ybd)
    h.vcycle(ybd, xbd)
    ok = [i for i in range(SMALL.nrhs) if i != 2]
    assert np.array_equal(xbd.cpu().numpy()[ok], xd.cpu().numpy()[ok])
    assert not np.isfinite(xbd.cpu().numpy()[2]).all()
    with pytest.raises(nmg.NmgError) as ei:
        h.solve(ybd, torch.zeros_like(ybd), max_cycles=2)
    assert ei.value.status == 5 and ei.value.report["fail_rhs"] == 2


@pytest.mark.parametrize("cfg_id,nrhs,cycles", [(2, 2, 2), (3, 1, 1), (4, 1, 1)])
def test_full_size_configs_subset(cfg_id, nrhs, cycles):
    """BASELINE configs 2-4 at full grid size on a seeded RHS subset: residual histories."""
    cfg = ni.CONFIGS[cfg_id].replace(nrhs=nrhs)
    f, W, H, h = _both(cfg, max_rhs=nrhs)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=nrhs)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=cycles)
    orc = O.solve(H, y, tol=1e-300, max_cycles=cycles, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("C,n,nrhs", [(32, 256, 3), (48, 128, 2), (48, 256, 1)])
def test_cnn_strip_kernels(C, n, nrhs):
    """BF16x3 column-strip CNN kernels (n % 128 == 0): several 128-pixel strips, y-split units
    (few RHS), the first/last rows and columns (zero padding), C = 32 and 48; the CNN alone
    (OP_CNN, no normalisation) and one smoothing step (norm + CNN + F')."""
    cfg = ni.CONFIGS[3 if C == 48 else 2].replace(n=n, levels=4 if n == 128 else 5, nrhs=nrhs)
    f, W, H, h = _both(cfg, max_rhs=nrhs)
    rng = np.random.default_rng(11)
    u = (rng.standard_normal((nrhs, n, n)) / n).astype(np.float32)
    out = torch.zeros(nrhs, n, n, device=DEV)
    h.debug_op(1, nmg.OP_CNN, T(u), out)
    ref = O.cnn_forward(H.weights[0], u.astype(np.float64))
    got = out.cpu().numpy()
    assert rel_l2(got, ref) < 1e-5
    # the pixels on both sides of every 128-pixel strip boundary (h finished from the strip-edge
    # records): per pixel, relative to the image's largest value
    edges = sorted({c for x0 in range(128, n, 128) for c in (x0 - 1, x0)} | {0, n - 1})
    err = np.abs(got[:, :, edges] - ref[:, :, edges]).max() / np.abs(ref).max()
    assert err < 1e-5, err
    b = (3.0 * rng.standard_normal((nrhs, n, n))).astype(np.float32)
    x0 = rng.standard_normal((nrhs, n, n)).astype(np.float32)
    xs = T(x0)
    h.debug_op(1, nmg.OP_SMOOTH, T(b), xs)
    s = np.sqrt((b.astype(np.float64) ** 2).sum(axis=(1, 2)))[:, None, None]
    hv = O.cnn_forward(H.weights[0], b / s) * s
    want = x0 + O.level_filter(H, 0, hv)
    assert rel_l2(xs.cpu().numpy() - x0, want - x0) < 1e-5


@pytest.mark.parametrize("cfg_id,n", [(2, 256), (4, 256), (3, 512)])
def test_outer_residual_2d_ozaki(cfg_id, n):
    """fp64 outer residual of the 2D path at n % 128 == 0 (two Ozaki int8 tcgen05 passes,
    T = X C^T then y - T B^T - alpha x) against the oracle's fp64 A x (1e-12, north_star)."""
    cfg = ni.CONFIGS[cfg_id].replace(n=n, levels=int(np.log2(n)) - 3, nrhs=3)
    f = ni.operator_factors(cfg)
    H = O.build_hierarchy(2, f, cfg.alpha, cfg.levels)
    h = nmg.Hierarchy(2, n, cfg.levels, cfg.alpha, f, max_rhs=3)
    rng = np.random.default_rng(6)
    y = rng.standard_normal((3, n, n))
    x = rng.standard_normal((3, n, n)) * np.array([1.0, 1e-3, 1e3])[:, None, None]
    r = torch.zeros(3, n, n, dtype=torch.float64, device=DEV)
    rr = torch.zeros(3, dtype=torch.float64, device=DEV)
    h.residual(T(y, torch.float64), T(x, torch.float64), r, rr)
    want = y - O.apply_A(H, 0, x)
    for b in range(3):
        assert rel_l2(r.cpu().numpy()[b], want[b]) < 1e-12, b
    nrm = np.sqrt((want ** 2).sum(axis=(1, 2))) / np.sqrt((y ** 2).sum(axis=(1, 2)))
    assert np.allclose(rr.cpu().numpy(), nrm, rtol=1e-12)


@pytest.mark.parametrize("nrhs", [37, 64])
def test_rhs_lanes_bitwise_2d(nrhs):
    """2D handles with max_rhs * n^2 <= 2^26 cycle their batch as two RHS lanes on forked streams
    (lane boundaries on even RHS, so the level filter's RHS pairs are the same); the result is
    bitwise the one-lane result, through the device entry and the lane-pipelined host entry."""
    cfg = SMALL.replace(nrhs=nrhs)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=nrhs)
    outs = []
    for lanes in (1, 0):
        h = gpu_hierarchy(cfg, f, W, max_rhs=64, tuning={"lanes": lanes})
        yd = T(y, torch.float64)
        xd = torch.zeros_like(yd)
        st = torch.cuda.Stream()
        for _ in range(3):                     # eager, capture, replay
            h.vcycle(yd, xd, st)
        torch.cuda.synchronize()
        outs.append(xd.cpu().numpy())
        xh = np.zeros_like(y)
        h.vcycles_host(np.ascontiguousarray(y), xh, 3, stream=st)
        outs.append(xh)
        h.close()
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
