"""GPU parity of the slab-sharded single-system mode (BASELINE config 4: the 2D
operator row-sharded over the ranks, nmg_create_hierarchy_slab).

One GPU is available here, so W ranks run as W host threads of this process, each with its own
stream and its own handle, exchanging data through the library's emulated communicator
(nmg_comm_create_emulated: host barriers + stream-ordered device copies, no device-side waits).
The per-rank program is the one a W-process NCCL run executes; only the transport differs.
Checks: residual histories against the fp64 oracle (north_star: 1e-3 relative), the fp64 outer
residual against the oracle (1e-12), the iterate against the unsharded GPU path (same kernels,
different summation order of the norms: rounding only), bitwise homogeneity (pin P10)."""
import threading

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
from paper_2603_01064_b200.parallel import join_slabs, split_slabs  # noqa: E402

DEV = torch.device("cuda:0")
# config 2's operator and smoother at n = 256 (W = 4: slabs of 64 rows at level 1, 32 at
# level 2, replicated from 64^2 down) and config 4's cos-modulated kernel (B != C)
CFG2 = ni.CONFIGS[2].replace(n=256, levels=5, nrhs=3)
CFG4 = ni.CONFIGS[4].replace(n=256, levels=5, nrhs=2, sigma=0.04)


def run_ranks(world, cfg, f, W, y, body):
    """Run body(rank, hierarchy, y_slab) on `world` emulated ranks (threads); returns results."""
    comms = nmg.Comm.emulated(world)
    ys = split_slabs(y, cfg.n, world)
    out = [None] * world
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, f, nu1=cfg.nu1, nu2=cfg.nu2,
                                  max_rhs=y.shape[0], comm=comms[r])
                for l, w in enumerate(W):
                    h.load_weights(l + 1, ni.cnn_arch(cfg), w)
                yd = torch.tensor(np.ascontiguousarray(ys[r]), dtype=torch.float64, device=DEV)
                out[r] = body(r, h, yd)
                torch.cuda.synchronize()
                h.close()
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    for c in comms:
        c.close()
    assert not errs, errs
    return out


@pytest.fixture(scope="module")
def prob2():
    f = ni.operator_factors(CFG2)
    W = weights_for(CFG2, "seed")
    y, _ = ni.make_rhs(CFG2, f, CFG2.alpha)
    return f, W, y, oracle_hierarchy(CFG2, f, W)


@pytest.fixture(scope="module")
def prob4():
    f = ni.operator_factors(CFG4)
    W = weights_for(CFG4, "seed")
    y, _ = ni.make_rhs(CFG4, f, CFG4.alpha)
    return f, W, y, oracle_hierarchy(CFG4, f, W)


def _solve_body(cycles):
    def body(r, h, yd):
        xd = torch.zeros_like(yd)
        rep = h.solve(yd, xd, tol=1e-300, max_cycles=cycles)
        return rep["history"], xd.cpu().numpy()
    return body


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_history_vs_oracle(world, prob2):
    f, W, y, H = prob2
    res = run_ranks(world, CFG2, f, W, y, _solve_body(3))
    orc = O.solve(H, y, tol=1e-300, max_cycles=3, freeze=False)
    for r in range(world):   # global relres: identical on every rank
        assert np.array_equal(res[r][0], res[0][0])
        ok, err = history_close(res[r][0], orc.history)
        assert ok, (world, r, err)


def test_slab_cos_kernel_vs_oracle_and_unsharded(prob4):
    """B != C (config 4's kernel): oracle histories, and the iterate against the unsharded path."""
    f, W, y, H = prob4
    res = run_ranks(4, CFG4, f, W, y, _solve_body(2))
    orc = O.solve(H, y, tol=1e-300, max_cycles=2, freeze=False)
    ok, err = history_close(res[0][0], orc.history)
    assert ok, err
    x_slab = join_slabs([res[r][1] for r in range(4)], CFG4.n)
    h = gpu_hierarchy(CFG4, f, W, max_rhs=y.shape[0])
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    h.solve(yd, xd, tol=1e-300, max_cycles=2)
    assert rel_l2(x_slab, xd.cpu().numpy().reshape(x_slab.shape)) < 1e-5


def test_slab_outer_residual_fp64(prob4):
    f, W, y, H = prob4
    x = np.random.default_rng(5).standard_normal(y.shape)
    xs = split_slabs(x, CFG4.n, 2)

    def body(r, h, yd):
        xd = torch.tensor(np.ascontiguousarray(xs[r]), dtype=torch.float64, device=DEV)
        rd = torch.zeros_like(yd)
        rr = torch.zeros(yd.shape[0], dtype=torch.float64, device=DEV)
        h.residual(yd, xd, rd, rr)
        return rd.cpu().numpy(), rr.cpu().numpy()

    res = run_ranks(2, CFG4, f, W, y, body)
    n = CFG4.n
    r = join_slabs([res[q][0] for q in range(2)], n)
    want = (y - O.apply_A(H, 0, x.reshape(-1, n, n)).reshape(y.shape)).reshape(r.shape)
    assert rel_l2(r, want) < 1e-12
    rel = np.linalg.norm(want, axis=1) / np.linalg.norm(y.reshape(r.shape), axis=1)
    assert np.allclose(res[0][1], rel, rtol=1e-12) and np.array_equal(res[0][1], res[1][1])


def test_slab_homogeneity_bitwise(prob2):
    """pin P10 on the sharded path: V(0, 4 y) = 4 V(0, y) bitwise (power-of-two scaling is exact
    through every kernel, and the rank sums run in a fixed order)."""
    f, W, y, H = prob2

    def body(r, h, yd):
        outs = []
        for s in (1.0, 4.0):
            ys = yd * s
            xd = torch.zeros_like(ys)
            h.vcycle(ys, xd)
            outs.append(xd.cpu().numpy() / s)
        return outs

    res = run_ranks(2, CFG2, f, W, y, body)
    for r in range(2):
        assert np.array_equal(res[r][0], res[r][1])


def test_slab_full_config4_w8_vs_unsharded():
    """BASELINE config 4 at full size (1024^2, 7 levels) over 8 emulated ranks (slabs of 128,
    64 and 32 rows; replicated from 128^2 down): one cycle equals the unsharded GPU path."""
    cfg = ni.CONFIGS[4].replace(nrhs=2)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=2)

    def body(r, h, yd):
        xd = torch.zeros_like(yd)
        h.vcycle(yd, xd)
        rr = torch.zeros(yd.shape[0], dtype=torch.float64, device=DEV)
        h.residual(yd, xd, None, rr)
        return xd.cpu().numpy(), rr.cpu().numpy()

    res = run_ranks(8, cfg, f, W, y, body)
    xs = join_slabs([res[r][0] for r in range(8)], cfg.n)
    h = gpu_hierarchy(cfg, f, W, max_rhs=2)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    h.vcycle(yd, xd)
    rr = torch.zeros(2, dtype=torch.float64, device=DEV)
    h.residual(yd, xd, None, rr)
    d = rel_l2(xs, xd.cpu().numpy().reshape(xs.shape))
    print("slab W=8 vs unsharded: x rel diff", d, "relres", res[0][1], rr.cpu().numpy())
    assert d < 1e-5
    assert np.allclose(res[0][1], rr.cpu().numpy(), rtol=1e-5)


@pytest.mark.parametrize("filt,nu1,nu2", [(False, 1, 1), (True, 1, 0), (True, 0, 1)])
def test_slab_variants_vs_unsharded(filt, nu1, nu2, prob2):
    """Cycle variants on the sharded path (filter off, no post-smoothing, no pre-smoothing) with
    an odd batch (the last level-filter pair has a zero partner): one cycle equals the unsharded
    GPU path (same kernels; rank sums in a fixed order)."""
    f, W, y, H = prob2
    cfg = CFG2.replace(nu1=nu1, nu2=nu2)
    comms = nmg.Comm.emulated(2)
    ys = split_slabs(y, cfg.n, 2)
    out, errs = [None, None], []

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                h = nmg.Hierarchy(2, cfg.n, cfg.levels, cfg.alpha, f, nu1=nu1, nu2=nu2, level_filter=filt,
                                  max_rhs=3, comm=comms[r])
                for l, w in enumerate(W):
                    h.load_weights(l + 1, ni.cnn_arch(cfg), w)
                yd = torch.tensor(np.ascontiguousarray(ys[r]), dtype=torch.float64, device=DEV)
                xd = torch.zeros_like(yd)
                h.vcycle(yd, xd)
                torch.cuda.synchronize()
                out[r] = xd.cpu().numpy()
                h.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    [t.start() for t in ts]
    [t.join(timeout=600) for t in ts]
    [c.close() for c in comms]
    assert not errs, errs
    xs = join_slabs(out, cfg.n)
    h = nmg.Hierarchy(2, cfg.n, cfg.levels, cfg.alpha, f, nu1=nu1, nu2=nu2, level_filter=filt, max_rhs=3)
    for l, w in enumerate(W):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    h.vcycle(yd, xd)
    assert rel_l2(xs, xd.cpu().numpy().reshape(xs.shape)) < 1e-5
