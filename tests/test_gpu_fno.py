"""GPU parity of the FNO smoother (NEXT-2; Appendix A, Table 6) against the fp64 oracle:
the raw network output (OP_CNN), one smoothing step (OP_SMOOTH: norm, FNO, level filter, update)
and whole-cycle residual histories with FNO smoothers on every level, 1D and 2D, Table-6
hyperparameters per level."""
import numpy as np
import pytest

import nmg_inputs as ni

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_01064_b200 as nmg  # noqa: E402
from oracle import nmg_oracle as O  # noqa: E402
from tests._setup import history_close  # noqa: E402

DEV = torch.device("cuda:0")
C1 = ni.CONFIGS[0]                                    # 1D n = 256, levels 256 / 128 smoothed
C2 = ni.CONFIGS[2].replace(n=64, levels=3, nrhs=3)    # 2D n = 64, levels 64 / 32 smoothed


def T(a, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def rel_rows(a, b):
    a = np.asarray(a, np.float64).reshape(a.shape[0], -1)
    b = np.asarray(b, np.float64).reshape(b.shape[0], -1)
    return np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)


def build(cfg, nrhs, simt=False):
    f = ni.operator_factors(cfg)
    Wf = ni.fno_weights_seed(cfg, seed=3)
    H = O.build_hierarchy(cfg.dim, f, cfg.alpha, cfg.levels, nu1=cfg.nu1, nu2=cfg.nu2)
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, f, nu1=cfg.nu1, nu2=cfg.nu2, max_rhs=nrhs,
                      tuning={"simt_fno": 1} if simt else None)
    for l, w in enumerate(Wf):
        arch = ni.fno_arch(cfg.dim, cfg.n >> l)
        O.load_weights(H, l + 1, O.fno_params(cfg.dim, *arch, w))
        h.load_fno_weights(l + 1, arch, w)
    return f, H, h


# default: the W-convolution on tcgen05 (3xTF32 implicit GEMM, fno_tc.cu); "-simt": the fp32 SIMT
# convolution kernels (nmg_tuning.simt_fno), which also serve the shapes the tensor-core kernel
# does not take
@pytest.fixture(scope="module", params=["1d", "2d", "1d-simt", "2d-simt"])
def setup(request):
    cfg = C1 if request.param.startswith("1d") else C2
    return (cfg,) + build(cfg, 4, simt=request.param.endswith("simt"))


def test_fno_forward_per_level(setup):
    cfg, f, H, h = setup
    rng = np.random.default_rng(7)
    for lvl in range(1, cfg.levels):
        n = cfg.n >> (lvl - 1)
        shape = (3,) + (n,) * cfg.dim
        u = rng.standard_normal(shape)
        u /= np.sqrt((u.reshape(3, -1) ** 2).sum(1)).reshape((3,) + (1,) * cfg.dim)
        out = torch.zeros(shape, device=DEV)
        h.debug_op(lvl, nmg.OP_CNN, T(u), out)
        want = O.fno_forward(H.weights[lvl - 1], u)
        assert rel_rows(out.cpu().numpy(), want).max() < 1e-5, lvl


def test_fno_smoothing_step(setup):
    cfg, f, H, h = setup
    rng = np.random.default_rng(8)
    n = cfg.n
    shape = (3,) + (n,) * cfg.dim
    b = 5.0 * rng.standard_normal(shape)
    x0 = rng.standard_normal(shape)
    xs = T(x0)
    h.debug_op(1, nmg.OP_SMOOTH, T(b), xs)
    b32 = b.astype(np.float32).astype(np.float64)
    s = np.sqrt((b32.reshape(3, -1) ** 2).sum(1)).reshape((3,) + (1,) * cfg.dim)
    hv = O.fno_forward(H.weights[0], b32 / s) * s
    want = O.level_filter(H, 0, hv)
    got = xs.cpu().numpy().astype(np.float64) - x0.astype(np.float32)
    # F' is a contraction (mask <= 1) that removes the large smooth part of h (here
    # ||h|| / ||F'(h)|| ~ 1e3 with the bias-dominated seeded FNO), so the fp32 error of h is
    # measured against ||h||: |F'(h_gpu) - F'(h)| <= |h_gpu - h|
    err = np.linalg.norm((got - want).reshape(3, -1), axis=1) / np.linalg.norm(hv.reshape(3, -1), axis=1)
    assert err.max() < 1e-5


def test_fno_cycle_history(setup):
    cfg, f, H, h = setup
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=3)
    yd = T(y, torch.float64)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=3)
    orc = O.solve(H, y, tol=1e-300, max_cycles=3, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("dim,n,nrhs,knob", [(1, 4096, 3, 0), (1, 512, 5, 0), (2, 256, 2, 0), (2, 128, 3, 0),
                                             (2, 16, 5, 0), (2, 128, 2, 2), (2, 128, 2, 1)])
def test_fno_forward_table6_sizes(dim, n, nrhs, knob):
    """Raw FNO output at the BASELINE level sizes (Table 6 rows: ks = 7 / 5 / 3, k up to 128; the
    tensor-core convolution's 1D tiles, the 2D row-halo kernel at n >= 128 and the 16 x 8 pixel boxes
    at n = 16, several tiles per image and tap shifts crossing the image border), per RHS against the
    oracle.  knob = nmg_tuning.simt_fno: 2 = the box kernel where the row-halo kernel would run,
    1 = the fp32 SIMT convolution."""
    base = ni.CONFIGS[1] if dim == 1 else ni.CONFIGS[2]
    levels = max(2, int(np.log2(n // (256 if dim == 1 else 16))) + 1)   # coarsest system <= 256 unknowns
    cfg = base.replace(n=n, levels=levels, nrhs=nrhs)
    f = ni.operator_factors(cfg)
    arch = ni.fno_arch(dim, n)
    w = ni.fno_weights_seed(cfg, seed=5)[0]
    h = nmg.Hierarchy(dim, n, levels, cfg.alpha, f, max_rhs=nrhs, tuning={"simt_fno": knob} if knob else None)
    h.load_fno_weights(1, arch, w)
    rng = np.random.default_rng(11)
    shape = (nrhs,) + (n,) * dim
    u = rng.standard_normal(shape)
    u /= np.sqrt((u.reshape(nrhs, -1) ** 2).sum(1)).reshape((nrhs,) + (1,) * dim)
    out = torch.zeros(shape, device=DEV)
    h.debug_op(1, nmg.OP_CNN, T(u), out)
    want = O.fno_forward(O.fno_params(dim, *arch, w), u)
    assert rel_rows(out.cpu().numpy(), want).max() < 1e-5
    h.close()


def test_fno_replaced_by_cnn_and_back():
    """Loading a CNN on an FNO level replaces it (and vice versa); graphs are re-captured."""
    cfg = C1
    f, H, h = build(cfg, 2)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=2)
    yd = T(y, torch.float64)
    W = ni.weights_seed(cfg)
    for l, w in enumerate(W):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    Hc = O.build_hierarchy(1, f, cfg.alpha, cfg.levels)
    for l, w in enumerate(W):
        O.load_weights(Hc, l + 1, ni.unflatten_params(cfg, w))
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-300, max_cycles=2)
    orc = O.solve(Hc, y, tol=1e-300, max_cycles=2, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err
