"""CPU checks of the level-wise smoother trainer (trainer/nmg_train.py, NEXT-1, Alg 5).

* Its differentiable transcription of the NMGF cycle equals the fp64 oracle's cycle (1D and
  2D, nu1/nu2 variants): the trainer and the oracle share no code, so this pins the trainer's
  forward pass (operators, transfers, Galerkin chain, masks, filter, CNN, coarse solve).
* The fine-grid loss masks m_l follow P:289-293 / P:405-409 (values at the band edges).
* Each level-wise loss L_l moves only theta_l (L_l(theta_l; {theta_k}_{k<l}), eq. loss_2_modified).
* A short run lowers every level's loss and the trained cycle converges on config 0.
"""
import math

import numpy as np
import pytest
import torch

import nmg_inputs as ni
from oracle import nmg_oracle as O
from trainer import nmg_train as T


def _oracle(cfg, f, W, nu1, nu2):
    H = O.build_hierarchy(cfg.dim, f, cfg.alpha, cfg.levels, nu1=nu1, nu2=nu2)
    for l, w in enumerate(W):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    return H


@pytest.mark.parametrize("which,nu1,nu2", [("1d", 1, 0), ("1d", 1, 1), ("2d", 1, 1), ("2d", 1, 0)])
def test_transcription_cycle_matches_oracle(which, nu1, nu2):
    cfg = ni.CONFIGS[0] if which == "1d" else ni.CONFIGS[2].replace(n=32, levels=3, nrhs=3)
    f = ni.operator_factors(cfg)
    W = ni.weights_seed(cfg)
    H = _oracle(cfg, f, W, nu1, nu2)
    lv = T.TorchLevels(cfg, f, cfg.alpha, "cpu", dtype=torch.float64)
    nets = [T.CNN(cfg, w, dtype=torch.float64) for w in W]
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=3)
    got = T.nmgf0(lv, nets, torch.tensor(y), nu1, nu2).numpy()
    want = O.nmgf_cycle(H, np.zeros_like(y), y)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-10


def test_export_folds_output_scale():
    """The 1/alpha output gain used during training folds exactly into the exported CNN."""
    cfg = ni.CONFIGS[0]
    w = ni.weights_seed(cfg)[0]
    net = T.CNN(cfg, w, out_scale=1e3, dtype=torch.float64)
    u = torch.randn(2, cfg.n, dtype=torch.float64)
    plain = T.CNN(cfg, net.export(), dtype=torch.float64)
    assert torch.allclose(net(u), plain(u), rtol=1e-6, atol=0)


def test_fine_masks_paper_values():
    """m_l on the finest grid: 1 at the band edge |phi| = pi/2^{l-1}, 0 at phi = 0 and
    outside the band; 2D: max(|phi1|, |phi2|) inside the box, 0 outside."""
    cfg = ni.CONFIGS[0].replace(n=16, levels=3)
    lv = T.TorchLevels(cfg, ni.operator_factors(cfg), cfg.alpha, "cpu", dtype=torch.float64)
    m1, m2 = lv.mask_fine[0].numpy(), lv.mask_fine[1].numpy()
    assert m1[0] == 0 and m1[8] == 1.0 and math.isclose(m1[4], math.sqrt(0.5))     # phi = pi, pi/2
    assert m2[4] == 1.0 and m2[8] == 0.0 and math.isclose(m2[2], math.sqrt(0.5))   # l = 2: edge pi/2
    c2 = ni.CONFIGS[2].replace(n=16, levels=3)
    lv2 = T.TorchLevels(c2, ni.operator_factors(c2), c2.alpha, "cpu", dtype=torch.float64)
    M2 = lv2.mask_fine[1].numpy()
    assert M2[4, 0] == 1.0 and M2[4, 8] == 0.0 and M2[0, 0] == 0.0


def test_level_losses_isolate_their_level():
    cfg = ni.CONFIGS[0]
    f = ni.operator_factors(cfg)
    lv = T.TorchLevels(cfg, f, cfg.alpha, "cpu", dtype=torch.float64)
    nets = [T.CNN(cfg, w, out_scale=1.0 / cfg.alpha, dtype=torch.float64) for w in ni.weights_seed(cfg)]
    rng = np.random.default_rng(3)
    x, y = T.data_generation(lv, nets, 4, 2, rng)
    losses = T.level_losses(lv, nets, x, y)
    for l, L_l in enumerate(losses):
        grads = torch.autograd.grad(L_l, [p for n in nets for p in n.parameters()], allow_unused=True,
                                    retain_graph=True)
        per = [grads[2 * len(nets[0].w) * k: 2 * len(nets[0].w) * (k + 1)] for k in range(len(nets))]
        for k, gk in enumerate(per):
            nz = any(g is not None and bool(torch.any(g != 0)) for g in gk)
            assert nz == (k == l), (l, k)


def test_short_training_converges_cfg0():
    torch.manual_seed(0)
    cfg = ni.CONFIGS[0]
    w, hist = T.train(cfg, cfg.alpha, ni.weights_seed(cfg), 150, seed=1, verbose=False)
    assert np.all(hist[-10:].mean(axis=0) < 0.5 * hist[:10].mean(axis=0))
    h = T.eval_solve(cfg, cfg.alpha, w, nrhs=4, max_cycles=40)
    assert np.nanmax(h[:, -1]) <= 1e-6


@pytest.mark.parametrize("dim", [1, 2])
def test_fno_module_matches_oracle(dim):
    """The trainer's FNO (torch.fft) equals the oracle's FNO (numpy loops over modes, Appendix A
    P:651-657) on the same flat Table-6 parameters, and export() folds the 1/alpha gain."""
    n = 64 if dim == 1 else 32
    cfg = ni.CONFIGS[0] if dim == 1 else ni.CONFIGS[2].replace(n=32, levels=3, nrhs=3)
    arch = ni.fno_arch(dim, n)
    cfg = cfg.replace(n=n)
    w = ni.fno_weights_seed(cfg, seed=5)[0]
    net = T.FNO(dim, n, w, out_scale=1e3, dtype=torch.float64)
    u = np.random.default_rng(1).standard_normal((2,) + (n,) * dim)
    want = O.fno_forward(O.fno_params(dim, *arch, w), u)
    assert np.abs(net(torch.tensor(u)).detach().numpy() - want).max() < 1e-10 * np.abs(want).max()
    plain = T.FNO(dim, n, net.export(), dtype=torch.float64)
    assert np.abs(plain(torch.tensor(u)).detach().numpy() - want).max() < 1e-5 * np.abs(want).max()


def test_fno_short_training_converges():
    """Level-wise training (Alg 5) of the FNO smoothers lowers the losses and the trained cycle
    converges on config 0 (the paper's own smoother, Appendix A)."""
    cfg = ni.CONFIGS[0]
    torch.manual_seed(0)
    w, hist = T.train(cfg, cfg.alpha, ni.fno_weights_seed(cfg), 40, arch="fno", verbose=False)
    hist = np.asarray(hist)
    assert np.all(hist[-5:].mean(0) < hist[:5].mean(0))
    h = T.eval_solve(cfg, cfg.alpha, w, nrhs=2, max_cycles=60, arch="fno")
    assert np.nanmax(h[:, -1]) < 1e-6
