"""GPU parity of cycle variants: nu2 = 0 (the paper's backslash cycle), filter off
(Alg 2), a single-level hierarchy (exact solve), nu1 = 2 / nu2 = 2, nu1 = 0,
the paper's own operator form G = K, and the SIMT/FFMA fallbacks."""
import os
import subprocess
import sys

import numpy as np
import pytest

import nmg_inputs as ni
from tests._setup import gpu_hierarchy, history_close, oracle_hierarchy, rel_l2, weights_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import nmg_oracle as O  # noqa: E402

DEV = torch.device("cuda:0")


def _run(cfg, kind="seed", level_filter=True, paper_form=False, cycles=4, tol=1e-300):
    f = ni.operator_factors(cfg, paper_form=paper_form)
    W = weights_for(cfg, kind)
    H = oracle_hierarchy(cfg, f, W, level_filter=level_filter)
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs, level_filter=level_filter)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=tol, max_cycles=cycles)
    orc = O.solve(H, y, tol=tol, max_cycles=cycles, freeze=tol > 1e-100)
    return rep, orc, xd.cpu().numpy()


@pytest.mark.parametrize("nu1,nu2", [(1, 0), (2, 2), (0, 1)])
def test_smoothing_counts_1d(nu1, nu2):
    cfg = ni.CONFIGS[0].replace(nu1=nu1, nu2=nu2)
    rep, orc, _ = _run(cfg)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_filter_off_1d():
    rep, orc, _ = _run(ni.CONFIGS[0], level_filter=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_single_level_is_exact_solve():
    """L = 1: each cycle is the coarse Cholesky solve.  The inner cycle's fp32 output limits one
    cycle to ~kappa * u_fp32; the fp64 correction-form outer iteration then refines it."""
    cfg = ni.CONFIGS[0].replace(n=64, levels=1, nrhs=3)
    rep, orc, x = _run(cfg, cycles=3)
    assert rep["history"][:, 1].max() < 1e-4
    assert rep["history"][:, 3].max() < 1e-10
    assert rel_l2(x, orc.x) < 1e-8


def test_paper_form_operator_1d():
    """A = alpha I + K instead of the BASELINE K^T K + alpha I."""
    cfg = ni.CONFIGS[0].replace(alpha=1e-2)
    rep, orc, _ = _run(cfg, paper_form=True)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_wlin_nu2_zero_converges_like_oracle():
    cfg = ni.CONFIGS[0].replace(nu2=0)
    rep, orc, _ = _run(cfg, kind="lin", cycles=60, tol=1e-6)
    assert rep["converged"].all() and orc.converged.all()
    assert np.abs(rep["cycles"] - orc.cycles).max() <= 1
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("nu1,nu2,filt", [(1, 0, True), (2, 1, False)])
def test_variants_2d(nu1, nu2, filt):
    cfg = ni.CONFIGS[2].replace(n=32, levels=2, nrhs=2, nu1=nu1, nu2=nu2)
    rep, orc, _ = _run(cfg, level_filter=filt, cycles=3)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


def test_paper_form_operator_2d():
    """hat A = alpha I (x) I + K (x) K."""
    cfg = ni.CONFIGS[2].replace(n=32, levels=2, nrhs=2, alpha=1e-2)
    rep, orc, _ = _run(cfg, paper_form=True, cycles=3)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("knob", ["simt_gemm", "ffma_cnn", "fp64_dmma", "no_graphs", "no_kron", "coarse_subst", "fused_coarse"])
@pytest.mark.parametrize("dim", [1, 2])
def test_fallback_kernels_match(knob, dim):
    """The alternative kernels selected by nmg_tuning (SIMT GEMM, FFMA CNNs, DMMA fp64 residual,
    eager launches, unfused Kronecker pair, Cholesky substitution at the coarsest level) agree
    with the oracle too."""
    if (knob == "no_kron" and dim == 1) or (knob == "fused_coarse" and dim == 2):
        pytest.skip("2D-only knob")
    cfg = ni.CONFIGS[0].replace(nrhs=2) if dim == 1 else ni.CONFIGS[2].replace(n=64, levels=3, nrhs=2)
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, "seed")
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=2, tuning={knob: 256 if knob == "fused_coarse" else 1})
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device="cuda")
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=3)
    orc = O.solve(H, y, tol=1e-300, max_cycles=3, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("kind,tol,cycles", [("seed", 1e-300, 10), ("lin", 1e-10, 120)])
def test_precision_fp64_cfg0(kind, tol, cycles):
    """NMG_PREC_FP64 (config 0's fp64 system, reading R14): the fused one-launch fp64 cycle.
    Histories match the fp64 oracle (the CNN's own arithmetic stays fp32, so over a long
    W_lin solve the histories move by ~kappa eps_32 / rho ~ 1e-4), and with W_lin
    the solve reaches 1e-10 -- far below what the fp32 inner cycle alone could -- at the oracle's
    cycle."""
    import paper_2603_01064_b200 as nmg
    cfg = ni.CONFIGS[0]
    f = ni.operator_factors(cfg)
    W = weights_for(cfg, kind)
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs, precision=nmg.PREC_FP64)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=tol, max_cycles=cycles)
    orc = O.solve(H, y, tol=tol, max_cycles=cycles, freeze=tol > 1e-100)
    ok, err = history_close(rep["history"], orc.history, tol=1e-3, floor=1e-12)
    assert ok, err
    if kind == "lin":
        assert rep["converged"].all() and np.array_equal(rep["cycles"], orc.cycles)
    # nmg_vcycle (graph-captured single launch) equals the solve's cycles
    x2 = torch.zeros_like(yd)
    for _ in range(3):
        h.vcycle(yd, x2)
    x3 = torch.zeros_like(yd)
    h.solve(yd, x3, tol=1e-300, max_cycles=3)
    assert torch.equal(x2, x3)


def test_anisotropic_operator_1d():
    """NEXT-3: the paper's anisotropic system A = alpha D + K, a(z) = 1 + 0.5 sin 2 pi z
    (PAPER.md:517-521), passed as G = K + alpha (D - I); histories vs the oracle."""
    cfg = ni.CONFIGS[0].replace(alpha=1e-2)
    f = ni.anisotropic_factors(cfg, cfg.alpha)
    W = weights_for(cfg, "seed")
    H = oracle_hierarchy(cfg, f, W)
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-300, max_cycles=4)
    orc = O.solve(H, y, tol=1e-300, max_cycles=4, freeze=False)
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err


@pytest.mark.parametrize("Lp", [5, 6])
def test_level_truncation_Lprime(Lp):
    """NEXT-3: test-time truncation L': smoothers trained on the 6-level
    config-1 hierarchy (W_train, alpha 1e-3), solved on the first L' levels with an exact solve
    at level L' (n_L' <= 256); converges to 1e-6 at the oracle's stopping cycles."""
    cfg = ni.CONFIGS[1].replace(alpha=1e-3)
    W = ni.weights_trained(cfg)
    if W is None:
        pytest.skip("no trained weights")
    c = cfg.replace(levels=Lp, nrhs=8)
    f = ni.operator_factors(c)
    Wl = W[:Lp - 1]
    H = oracle_hierarchy(c, f, Wl)
    h = gpu_hierarchy(c, f, Wl, max_rhs=8)
    y, _ = ni.make_rhs(c, f, c.alpha, nrhs=8)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-6, max_cycles=60)
    orc = O.solve(H, y, tol=1e-6, max_cycles=60)
    assert orc.converged.all() and rep["converged"].all()
    ok, err = history_close(rep["history"], orc.history)
    assert ok, err
    assert np.abs(rep["cycles"] - orc.cycles).max() <= 1


@pytest.mark.parametrize("dim", [1, 2])
def test_weight_reload_matches_fresh_handle(dim):
    """Reloading a level's smoother weights replaces them: the captured cycle graphs (which bake in
    weight pointers, tensor maps and by-value weights) are dropped, so cycles after the reload are
    bitwise those of a fresh handle created with the new weights (include/nmg.h,
    nmg_load_smoother_weights: "loading a level twice replaces it")."""
    cfg = ni.CONFIGS[0] if dim == 1 else ni.CONFIGS[2].replace(n=64, levels=3, nrhs=3)
    f = ni.operator_factors(cfg)
    W1, W2 = ni.weights_seed(cfg, seed=0), ni.weights_seed(cfg, seed=7)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    h = gpu_hierarchy(cfg, f, W1, max_rhs=cfg.nrhs)
    x1 = torch.zeros_like(yd)
    for _ in range(3):                         # eager run, graph capture, replay
        h.vcycle(yd, x1)
    for l, w in enumerate(W2):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    x2 = torch.zeros_like(yd)
    for _ in range(3):
        h.vcycle(yd, x2)
    hf = gpu_hierarchy(cfg, f, W2, max_rhs=cfg.nrhs)
    x3 = torch.zeros_like(yd)
    for _ in range(3):
        hf.vcycle(yd, x3)
    torch.cuda.synchronize()
    assert torch.equal(x2, x3)
    assert not torch.equal(x1, x2)


def test_divergence_check_is_opt_in():
    """SPEC.md:545 rule behind desc.divergence_check: a smoother that overshoots (W_seed scaled by 10:
    the 3-layer ReLU network's output grows 1000x) drives relres above 10x its initial value for 5
    consecutive cycles -> nmg_solve returns NMG_ERR_DIVERGED; without the flag the same solve runs
    its max_cycles and reports the growing history."""
    import paper_2603_01064_b200 as nmg
    cfg = ni.CONFIGS[0]
    f = ni.operator_factors(cfg)
    W = [10.0 * w for w in ni.weights_seed(cfg)]
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    yd = torch.tensor(y, dtype=torch.float64, device=DEV)
    h = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs)
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-6, max_cycles=6)
    hist = np.asarray(rep["history"])
    assert np.all(hist[:, -1] > 10.0 * hist[:, 0])
    hd = gpu_hierarchy(cfg, f, W, max_rhs=cfg.nrhs, divergence_check=True)
    with pytest.raises(nmg.NmgError) as e:
        hd.solve(yd, torch.zeros_like(yd), tol=1e-6, max_cycles=20)
    assert e.value.status == 9          # NMG_ERR_DIVERGED
