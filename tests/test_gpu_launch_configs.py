"""GPU parity at the benchmark's exact launch configurations (bench.py): full BASELINE batches on
handles sized like the bench's (1D: max_rhs 1024 -> four RHS lanes, 256-wide multicast FP16x3
GEMM tiles, Ozaki fp64 residual; 2D: the 8-RHS seeded pool tiled to the full batch, the strip-
kernel CNN in RHS chunks, Ozaki 2D residual, Kronecker applies).

Expected values: the fp64 oracle, precomputed by tools/make_oracle_goldens.py (calls only
oracle/ and nmg_inputs) into tests/golden/oracle_*.npz.  Tolerances (BASELINE.json north_star):
per-operator 1e-5 relative L2 PER RHS, residual histories 1e-3 relative until 1e-6, stopping
cycles equal (+-1 only when the oracle residual is within 1e-3 of the tolerance, reading R13).
"""
import os

import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, history_close, oracle_hierarchy, weights_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_01064_b200 as nmg  # noqa: E402
from oracle import nmg_oracle as O  # noqa: E402

DEV = torch.device("cuda:0")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CFG1 = ni.CONFIGS[1]


def T(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def rel_rows(a, b):
    """Relative L2 error of every RHS (row) separately."""
    a = np.asarray(a, np.float64).reshape(a.shape[0], -1)
    b = np.asarray(b, np.float64).reshape(b.shape[0], -1)
    nb = np.linalg.norm(b, axis=1)
    return np.linalg.norm(a - b, axis=1) / np.where(nb > 0, nb, 1.0)


def gold(name):
    return np.load(os.path.join(GOLD, name))


@pytest.fixture(scope="module")
def cfg1_bench():
    """The bench's config-1 handle: 1024 RHS, default lanes (four lanes of 256 RHS)."""
    f = ni.operator_factors(CFG1)
    W = weights_for(CFG1, "seed")
    return f, W, oracle_hierarchy(CFG1, f, W), gpu_hierarchy(CFG1, f, W, max_rhs=CFG1.nrhs)


@pytest.mark.parametrize("lvl", [1, 2])
def test_cfg1_operator_full_batch_per_rhs(cfg1_bench, lvl):
    """OP_APPLY / OP_RESIDUAL with the full 1024-RHS batch: level 1 runs the 256-wide FP16x3 GEMM
    with the operator tile multicast over CTA pairs (tc_gemm_kernel<256, f16, MC>), level 2 the
    64-wide tiles; every RHS within 1e-5 on its own."""
    _, _, H, h = cfg1_bench
    n = CFG1.n >> (lvl - 1)
    rng = np.random.default_rng(40 + lvl)
    x = rng.standard_normal((1024, n)).astype(np.float32)
    x *= np.logspace(-3, 3, 1024, dtype=np.float32)[:, None]        # per-RHS scales (per-row f16 split)
    y = rng.standard_normal((1024, n)).astype(np.float32)
    want = O.apply_A(H, lvl - 1, x.astype(np.float64))
    out = torch.zeros(1024, n, device=DEV)
    h.debug_op(lvl, nmg.OP_APPLY, T(x), out)
    assert rel_rows(out.cpu().numpy(), want).max() < 1e-5
    yy = y * np.abs(want).max(axis=1, keepdims=True).astype(np.float32)
    r = T(yy)
    h.debug_op(lvl, nmg.OP_RESIDUAL, T(x), r)
    assert rel_rows(r.cpu().numpy(), yy - want).max() < 1e-5


@pytest.mark.parametrize("alpha", ni.ALPHAS[1])
def test_cfg1_full_batch_wseed_alpha_sweep(alpha):
    """The bench's config-1 launch (1024 RHS, four lanes, Ozaki residual) for every alpha of the
    sweep: 10 W_seed cycles; 16 sampled RHS (lane edges 255/256, 511/512, 767/768 included)
    against the oracle's histories."""
    cfg = CFG1.replace(alpha=alpha)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs)
    y, _ = ni.make_rhs(cfg, f, alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=cfg.cycles)
    g = gold("oracle_cfg1_wseed.npz")
    idx = g["idx"]
    ok, err = history_close(rep["history"][idx], g[f"hist_{alpha:g}"])
    assert ok, err
    h.close()


@pytest.mark.parametrize("alpha", [1e-2, 1e-3])
def test_cfg1_wlin_solve_stopping_cycles(alpha):
    """RHS solved to 1e-6 (the bench's `solve` figure) with the converging W_lin stand-in:
    each sampled RHS stops at the oracle's cycle (+-1 only per reading R13) and its history
    matches until 1e-6."""
    cfg = CFG1.replace(alpha=alpha)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "lin")
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs)
    y, _ = ni.make_rhs(cfg, f, alpha)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-6, max_cycles=100)
    assert rep["converged"].all()
    g = gold("oracle_cfg1_wlin.npz")
    idx = g["idx"]
    oc, oh = g[f"cycles_{alpha:g}"], g[f"hist_{alpha:g}"]
    assert g[f"conv_{alpha:g}"].all()
    ok, err = history_close(rep["history"][idx], oh)
    assert ok, err
    for k, b in enumerate(idx):
        d = abs(int(rep["cycles"][b]) - int(oc[k]))
        if d:
            c = min(int(rep["cycles"][b]), int(oc[k]))
            assert d == 1 and abs(oh[k, c] - 1e-6) <= 1e-3 * 1e-6, (b, rep["cycles"][b], oc[k])
    h.close()


POOL = {"cfg2": (2, 1e-3), "cfg3_a1e-3": (3, 1e-3), "cfg3_a1e-4": (3, 1e-4), "cfg4": (4, 1e-4)}


@pytest.mark.parametrize("key", list(POOL))
def test_2d_bench_batch_tiled_pool(key):
    """The bench's 2D launch: the configuration's full batch (256 / 2048 / 32 RHS) built by tiling
    the 8-RHS seeded pool, on a handle with max_rhs = batch (RHS chunks of the strip CNN, lanes
    where the bench has them).  3 cycles; every batch RHS is bitwise its pool member's result
    (per-RHS independence), and the pool members' histories match the oracle's."""
    cid, alpha = POOL[key]
    cfg = ni.CONFIGS[cid].replace(alpha=alpha)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    B = cfg.nrhs
    pool, _ = ni.make_rhs(cfg, f, alpha, nrhs=8, start=0)
    y = np.ascontiguousarray(np.concatenate([pool] * (-(-B // 8)))[:B])
    h = gpu_hierarchy(cfg, f, W, max_rhs=B)
    yd = T(y, torch.float64)
    del y
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=3)
    hist = rep["history"]
    x = xd.view(B, -1)
    for b in range(8, B):
        assert np.array_equal(hist[b], hist[b % 8]), b
    for b in range(8, B, max(1, B // 64)):
        assert torch.equal(x[b], x[b % 8]), b
    g = gold("oracle_2d_pool.npz")[f"hist_{key}"]
    ok, err = history_close(hist[:g.shape[0]], g)
    assert ok, err
    h.close()
    del xd, yd
    torch.cuda.empty_cache()


def test_coarse_substitution_cfg1(cfg1_bench):
    """tuning.coarse_subst (Cholesky forward/back substitution, the north-star form of the
    coarsest solve) at config 1: same histories as the explicit-inverse default."""
    f, W, H, _ = cfg1_bench
    h = gpu_hierarchy(CFG1.replace(nrhs=4), f, W, max_rhs=4, tuning={"coarse_subst": 1})
    y, _ = ni.make_rhs(CFG1, f, CFG1.alpha, nrhs=4)
    yd = T(y, torch.float64)
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-300, max_cycles=4)
    orc = O.solve(H, y, tol=1e-300, max_cycles=4, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def _wtrain_keys():
    p = os.path.join(GOLD, "oracle_wtrain.npz")
    if not os.path.exists(p):
        return []
    with np.load(p) as z:
        return sorted(k[len("cycles_"):] for k in z.files if k.startswith("cycles_"))


@pytest.mark.parametrize("key", _wtrain_keys())
def test_wtrain_solve_matches_oracle(key):
    """The trained smoothers W_train (trainer/nmg_train.py, Alg 5) at the bench's launch
    configuration (full batch; 2D: the tiled pool): the oracle converged on its sample
    (tools/make_oracle_goldens.py), every GPU RHS converges to 1e-6 and the sampled RHS stop at
    the oracle's cycle.

    Tolerance: the inner cycle is
    fp32-accurate (per-operator error eps <= 1e-5, north star), so each cycle's correction
    carries an error whose residual image is up to kappa eps ||r_k||, kappa = (1 + alpha) / alpha
    (A's eigenvalues lie in [alpha, 1 + alpha]); relative to ||r_{k+1}|| = rho ||r_k|| that is
    kappa eps / rho.  Histories must agree to max(1e-3, kappa eps / rho) with rho the oracle's
    mean per-cycle reduction (1e-3 where the problem is well conditioned), stopping cycles to
    +-max(1, 5 %)."""
    name, a = key.rsplit("_a", 1)
    alpha = float(a)
    cid = [c for c, v in ni.CONFIGS.items() if v.name == name][0]
    cfg = ni.CONFIGS[cid].replace(alpha=alpha)
    W = ni.weights_trained(cfg)
    assert W is not None
    g = gold("oracle_wtrain.npz")
    oc, oh = g[f"cycles_{key}"], g[f"hist_{key}"]
    assert g[f"conv_{key}"].all()
    f = ni.operator_factors(cfg)
    B = cfg.nrhs
    kw = {}
    if cid == 0:   # all 8 RHS, in the bench's launch configuration (the fused fp64 cycle)
        import paper_2603_01064_b200 as nmg
        y, _ = ni.make_rhs(cfg, f, alpha)
        idx = list(range(B))
        kw = {"precision": nmg.PREC_FP64}
    elif cfg.dim == 1:
        y, _ = ni.make_rhs(cfg, f, alpha)
        idx = list(gold("oracle_cfg1_wseed.npz")["idx"])
    else:
        pool, _ = ni.make_rhs(cfg, f, alpha, nrhs=8, start=0)
        y = np.ascontiguousarray(np.concatenate([pool] * (-(-B // 8)))[:B])
        idx = list(range(len(oc)))
    h = gpu_hierarchy(cfg, f, W, max_rhs=B, **kw)
    yd = T(y, torch.float64)
    del y
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-6, max_cycles=150)
    assert rep["converged"].all()
    rho = float(np.mean([(1e-6 / oh[k, 0]) ** (1.0 / max(1, oc[k])) for k in range(len(oc))]))
    tol = max(1e-3, (1.0 + alpha) / alpha * 1e-5 / rho)
    hg = rep["history"][idx]
    m = np.isfinite(oh) & (oh >= 1e-6)
    dev = np.where(m, np.abs(hg - oh) / np.where(m, oh, 1.0), 0.0)
    print(key, f"rho {rho:.3f} tol {tol:.2e} max history deviation {dev.max():.2e}; cycles gpu",
          rep["cycles"][idx].tolist(), "oracle", oc.tolist())
    assert dev.max() <= tol
    for k, b in enumerate(idx):
        assert abs(int(rep["cycles"][b]) - int(oc[k])) <= max(1, int(np.ceil(0.05 * oc[k]))), (b, rep["cycles"][b], oc[k])
    h.close()


@pytest.mark.parametrize("name,cid,alpha", [("cfg1_a1e-4", 1, 1e-4), ("cfg1_a1e-3", 1, 1e-3), ("cfg2_a1e-3", 2, 1e-3)])
def test_wtrain_smoother_per_level(name, cid, alpha):
    """The FP16x3 tensor-core CNN with TRAINED weights (large output gains, activations far from
    the power-of-two scales' worst-case bounds): OP_CNN and OP_SMOOTH at every smoothed level
    within 1e-5 per RHS (the smoothing step measured against ||h||: F' is a contraction)."""
    cfg = ni.CONFIGS[cid].replace(alpha=alpha)
    W = ni.weights_trained(cfg)
    if W is None:
        pytest.skip("no trained weights")
    f = ni.operator_factors(cfg)
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=8)
    rng = np.random.default_rng(12)
    for lvl in range(1, cfg.levels):
        n = cfg.n >> (lvl - 1)
        shape = (4,) + (n,) * cfg.dim
        b = rng.standard_normal(shape) * np.logspace(-2, 2, 4).reshape((4,) + (1,) * cfg.dim)
        b = b.astype(np.float32).astype(np.float64)
        s = np.sqrt((b.reshape(4, -1) ** 2).sum(1)).reshape((4,) + (1,) * cfg.dim)
        u = b / s
        out = torch.zeros(shape, device=DEV)
        h.debug_op(lvl, nmg.OP_CNN, T(u), out)
        want = O.cnn_forward(H.weights[lvl - 1], u.astype(np.float32).astype(np.float64))
        e1 = rel_rows(out.cpu().numpy(), want).max()
        x0 = rng.standard_normal(shape).astype(np.float32)
        xs = T(x0)
        h.debug_op(lvl, nmg.OP_SMOOTH, T(b), xs)
        hv = O.cnn_forward(H.weights[lvl - 1], u) * s
        wantx = O.level_filter(H, lvl - 1, hv)
        got = xs.cpu().numpy().astype(np.float64) - x0
        err = np.linalg.norm((got - wantx).reshape(4, -1), axis=1) / np.linalg.norm(hv.reshape(4, -1), axis=1)
        print(name, "level", lvl, "cnn", e1, "smooth", err.max())
        assert e1 < 1e-5, ("cnn", lvl, e1)
        assert err.max() < 1e-5, ("smooth", lvl, err)
    h.close()
