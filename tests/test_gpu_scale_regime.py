"""FP16x3 scale regime of the tensor-core CNN smoothers.

The split-precision CNN kernels (smooth1d_f16.cu, conv_strip.cu) multiply v S = hi + lo in f16
with a power-of-two scale S per layer chosen at weight-load time from a worst-case activation
bound.  Accuracy then depends on how far the real activations sit below that
bound: f16 has 5 exponent bits, so activations many decades below it lose hi/lo bits to
subnormals.  These cases push that regime against the fp64 oracle, per RHS, at the smoothing
step's 1e-5 (north_star's fp32-accurate per-operator bound):
  * zero biases (a1 = ReLU(w0 * u) scales with u exactly, nothing lifts it off zero);
  * per-output-channel weight magnitudes spread over three decades (the bound is set by the
    largest channel, the small channels sit 10^3 below it: the library lifts such channels by
    an exactly equivalent power-of-two rebalancing at weight load, nmg_api.cu balance_cnn);
  * RHS with a wide dynamic range: a localized spike over 1e-6-level noise, and entries with
    log-uniform magnitudes over six decades (u = b / ||b|| then has most entries far below 1).
Smoothing step per PAPER.md Alg 3 line 2 with F' of P:305 (1D) / P:415 (2D).
"""
import math

import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, oracle_hierarchy

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_01064_b200 as nmg  # noqa: E402
from oracle import nmg_oracle as O  # noqa: E402

DEV = torch.device("cuda:0")


def _spread_weights(cfg, seed):
    """Kaiming-uniform weights whose output channels are scaled by 10^U(-3, 0), zero biases
    (one flat vector per smoothed level, the layout of ni.flatten_params)."""
    rng = np.random.default_rng(seed)
    out = []
    for _lvl in range(1, cfg.levels):
        layers = []
        for ws, bs in ni.layer_shapes(cfg):
            fan_in = int(np.prod(ws[1:]))
            wb = math.sqrt(6.0 / fan_in)
            w = rng.uniform(-wb, wb, size=ws)
            w *= (10.0 ** rng.uniform(-3.0, 0.0, size=ws[0])).reshape((ws[0],) + (1,) * (len(ws) - 1))
            layers.append((w, np.zeros(bs)))
        out.append(ni.flatten_params(layers))
    return out


def _wide_rhs(rng, shape):
    """RHS 0: a spike over 1e-6 noise; RHS 1: log-uniform magnitudes over six decades with random
    signs; the rest standard normal."""
    b = rng.standard_normal(shape)
    flat = b.reshape(shape[0], -1)
    flat[0] *= 1e-6
    flat[0, flat.shape[1] // 3] = 1.0
    if shape[0] > 1:
        flat[1] = np.sign(rng.standard_normal(flat.shape[1])) * 10.0 ** rng.uniform(-6.0, 0.0, flat.shape[1])
    return flat.reshape(shape).astype(np.float32)


def _per_rhs_rel(got, want):
    g = got.reshape(got.shape[0], -1).astype(np.float64)
    w = want.reshape(want.shape[0], -1)
    return np.linalg.norm(g - w, axis=1) / np.linalg.norm(w, axis=1)


CASES = [
    # (config, n, levels, nrhs): 1D n = 4096 runs smooth1d_f16 at the cfg 1 level-1 size, 2D runs
    # the column-strip kernels at C = 32 (cfg 2) and C = 48 (cfg 3)
    (1, 4096, 6, 4),
    (1, 256, 3, 3),
    (2, 256, 5, 3),
    (3, 128, 4, 3),
]


@pytest.mark.parametrize("cid,n,levels,nrhs", CASES)
def test_smoothing_step_scale_regime(cid, n, levels, nrhs):
    cfg = ni.CONFIGS[cid].replace(n=n, levels=levels, nrhs=nrhs)
    f = ni.operator_factors(cfg)
    W = _spread_weights(cfg, seed=17 + cid)
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=nrhs)
    rng = np.random.default_rng(23)
    shape = (nrhs, n) if cfg.dim == 1 else (nrhs, n, n)
    b = _wide_rhs(rng, shape)
    x0 = np.zeros(shape, np.float32)   # the update alone (no fp32 cancellation against x0)
    xs = torch.tensor(x0, device=DEV)
    h.debug_op(1, nmg.OP_SMOOTH, torch.tensor(b, device=DEV), xs)
    b64 = b.astype(np.float64)
    axes = tuple(range(1, b.ndim))
    s = np.sqrt((b64 ** 2).sum(axis=axes)).reshape((nrhs,) + (1,) * (b.ndim - 1))
    hv = O.cnn_forward(H.weights[0], b64 / s) * s
    want = O.level_filter(H, 0, hv)
    err = _per_rhs_rel(xs.cpu().numpy() - x0, want)
    assert err.max() < 1e-5, err


@pytest.mark.parametrize("cid,n,levels,nrhs", CASES)
def test_cnn_scale_regime(cid, n, levels, nrhs):
    """The CNN alone (OP_CNN, no normalisation) on a unit-norm input with a wide dynamic range.

    The debug entry accepts un-normalised inputs |u| <= 16, so its split scales sit 2^4 below the
    product path's (|u| <= 1 after the normalisation): 16x the FP16x3 rounding floor, hence
    1e-5 x 16 here.  The product path (the smoothing step above) holds 1e-5."""
    cfg = ni.CONFIGS[cid].replace(n=n, levels=levels, nrhs=nrhs)
    f = ni.operator_factors(cfg)
    W = _spread_weights(cfg, seed=29 + cid)
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=nrhs)
    rng = np.random.default_rng(31)
    shape = (nrhs, n) if cfg.dim == 1 else (nrhs, n, n)
    u = _wide_rhs(rng, shape).astype(np.float64)
    u /= np.sqrt((u ** 2).reshape(nrhs, -1).sum(axis=1)).reshape((nrhs,) + (1,) * (u.ndim - 1))
    u = u.astype(np.float32)
    out = torch.zeros(shape, device=DEV)
    h.debug_op(1, nmg.OP_CNN, torch.tensor(u, device=DEV), out)
    want = O.cnn_forward(H.weights[0], u.astype(np.float64))
    err = _per_rhs_rel(out.cpu().numpy(), want)
    assert err.max() < 16e-5, err


@pytest.mark.parametrize("cid,n,levels,nrhs", [(1, 256, 3, 3), (2, 64, 3, 3)])
def test_balance_is_exact_on_fp32_kernels(cid, n, levels, nrhs):
    """The hidden-channel rebalancing (powers of two, ReLU homogeneity) is an exactly equivalent
    network: on the plain fp32 FFMA kernels (nmg_tuning.ffma_cnn) the balanced and the as-given
    weights give bitwise the same CNN output."""
    cfg = ni.CONFIGS[cid].replace(n=n, levels=levels, nrhs=nrhs)
    f = ni.operator_factors(cfg)
    W = _spread_weights(cfg, seed=41 + cid)
    rng = np.random.default_rng(43)
    shape = (nrhs, n) if cfg.dim == 1 else (nrhs, n, n)
    u = torch.tensor(_wide_rhs(rng, shape), device=DEV)
    outs = []
    for nb in (0, 1):
        h = gpu_hierarchy(cfg, f, W, max_rhs=nrhs, tuning={"ffma_cnn": 1, "no_balance": nb})
        out = torch.zeros(shape, device=DEV)
        h.debug_op(1, nmg.OP_CNN, u, out)
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
