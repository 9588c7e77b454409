#!/usr/bin/env python
"""Level-wise training of the CNN neural smoothers.

Implements PAPER.md Alg 5 "Training of neural smoothers" for the BASELINE CNN
architecture (reading R7), with the filtered level-wise losses of eq. loss_2_modified
(1D) and eq. loss_3 (2D), Adam and the alpha curriculum
(P:477).  This is a TOOL, not the solve path: gradients come from PyTorch autograd on its own
differentiable transcription of the cycle below; the rollout of DataGeneration runs
through the C ABI (nmg_vcycle of libnmg.so) when a GPU is present ("nmg"), or through the same
transcription ("torch", CPU runs and tests).  It shares no code with oracle/ (the tests pin
its cycle against the oracle).

Per epoch (Alg 5):
  1. DataGeneration: x_i ~ N(0, I) i.i.d. per grid point (the paper's "given distribution" is
     unstated; white noise carries every frequency band), y_i = A x_i, k ~ U{1..K}, then k
     times x_i <- x_i - NMGF(0, y_i), y_i <- A x_i (the error after one more cycle and its
     residual: reading R20 of the erratum in the paper's rollout line).  Samples are scaled to
     unit ||x_i|| (the cycle is positively 1-homogeneous, pin P10, so this only balances the
     batch).
  2. Evaluate NMGF(0, y_i) with nu1 = 1, nu2 = 0 (Alg 3 / Alg 4 as trained in the paper):
       level l: b_l = y_l, h_l = N_l(b_l / ||b_l||) ||b_l||, x_l = F'_l(h_l),
                y_{l+1} = I_l^{l+1}(y_l - A_l x_l).
  3. L_l = 1/N sum_i || F_l( x_i - sum_{k<l} I_k^1 F'_k(h_k) - I_l^1 h_l ) ||^2 with the fine-grid
     mask F_l(v) = m_l (.) DFT_1(v), m_l = sqrt(|phi| / (pi / 2^{l-1})) on the band
     |phi| <= pi / 2^{l-1} sampled on n_1 points (reading R21; 2D: max(|phi1|,|phi2|)
     inside the box).  Each L_l only moves theta_l: the inputs b_l and the coarser
     terms of the finer levels are detached (L_l(theta_l; {theta_k}_{k<l})).
  4. theta_l <- Adam step on grad L_l for every l.

Output scale: the network is trained as h = (1/alpha) N(u) ||b||, the constant 1/alpha folded
into the last layer's weight and bias on export (an exactly equivalent CNN of the R7 family), so
the optimiser does not have to grow a 1/alpha gain from a Kaiming start.

Usage (GPU box):  python trainer/nmg_train.py --config 1 --alphas 1e-2 1e-3 1e-4 --epochs 1500
writes nmg_inputs/trained/W_train_<cfg>_a<alpha>.npz (flat fp32 vectors, state_dict order).
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time
from typing import List, Optional

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import nmg_inputs as ni  # noqa: E402

OUT_DIR = os.path.join(ROOT, "nmg_inputs", "trained")


# ------------------------------------------------------------------------------------------
# Problem hierarchy in torch (Galerkin chain P:160, transfers reading R4, masks reading R5)
# ------------------------------------------------------------------------------------------
def interp_np(n_c: int) -> np.ndarray:
    """Cell-centred linear interpolation P (n_f x n_c), reading R4: fine i takes 3/4 of
    coarse i >> 1 and 1/4 of its other neighbour (clamped at the ends)."""
    n_f = 2 * n_c
    P = np.zeros((n_f, n_c))
    for i in range(n_f):
        j = i >> 1
        k = min(max(j + (1 if i & 1 else -1), 0), n_c - 1)
        P[i, j] += 0.75
        P[i, k] += 0.25
    return P


class TorchLevels:
    """Operators of every level: 1D dense A_l; 2D Kronecker factors (B_l, C_l, Q_l) with
    A_l X = C X B^T + alpha Q X Q^T on the column-major X, i.e. B arr C^T +
    alpha Q arr Q^T on the row-major [i2][i1] array arr."""

    def __init__(self, cfg, factors, alpha: float, device, dtype=torch.float32):
        self.cfg, self.dim, self.L, self.alpha = cfg, cfg.dim, cfg.levels, alpha
        self.dev, self.dt = device, dtype
        ns = [cfg.n >> l for l in range(cfg.levels)]
        self.ns = ns
        t = lambda a: torch.tensor(a, dtype=dtype, device=device)   # noqa: E731
        Ps = [interp_np(ns[l + 1]) for l in range(self.L - 1)]
        self.P = [t(P) for P in Ps]
        self.R = [t(0.5 * P.T) for P in Ps]
        if self.dim == 1:
            A = np.array(factors[0], np.float64) + alpha * np.eye(cfg.n)
            self.A = [t(A)]
            for l in range(self.L - 1):
                A = 0.5 * Ps[l].T @ A @ Ps[l]
                self.A.append(t(A))
            Ac = A
        else:
            B, C, Q = (np.array(factors[0], np.float64), np.array(factors[1], np.float64), np.eye(cfg.n))
            self.B, self.C, self.Q = [t(B)], [t(C)], [t(Q)]
            for l in range(self.L - 1):
                B, C, Q = (0.5 * Ps[l].T @ M @ Ps[l] for M in (B, C, Q))
                self.B.append(t(B)); self.C.append(t(C)); self.Q.append(t(Q))
            Ac = np.kron(B, C) + alpha * np.kron(Q, Q)          # index i1 + n i2 = flat [i2][i1]
        self.Ainv = t(np.linalg.inv(Ac))
        self.mask_level = [t(self._level_mask(n)) for n in ns[:-1]]
        self.mask_fine = [t(self._fine_mask(l + 1)) for l in range(self.L - 1)]

    # --- masks
    def _level_mask(self, n):
        """m'_l in natural DFT order: sqrt(2 min(k, n-k) / n) (1D), sqrt(max(a(k1), a(k2))) (2D)."""
        a = 2.0 * np.minimum(np.arange(n), n - np.arange(n)) / n
        return np.sqrt(a) if self.dim == 1 else np.sqrt(np.maximum(a[:, None], a[None, :]))

    def _fine_mask(self, l):
        """m_l on the finest grid (n_1 points, reading R21): |phi_k| = 2 pi min(k, n-k) / n."""
        n = self.ns[0]
        q = 2.0 ** l * np.minimum(np.arange(n), n - np.arange(n)) / n     # |phi| / (pi / 2^{l-1})
        if self.dim == 1:
            return np.where(q <= 1.0, np.sqrt(q), 0.0)
        inside = (q[:, None] <= 1.0) & (q[None, :] <= 1.0)
        return np.where(inside, np.sqrt(np.maximum(q[:, None], q[None, :])), 0.0)

    # --- operators (batched, RHS-major)
    def apply(self, l, X):
        if self.dim == 1:
            return X @ self.A[l].T
        return self.B[l] @ X @ self.C[l].T + self.alpha * (self.Q[l] @ X @ self.Q[l].T)

    def restrict(self, l, X):
        return X @ self.R[l].T if self.dim == 1 else self.R[l] @ X @ self.R[l].T

    def interpolate(self, l, X):
        return X @ self.P[l].T if self.dim == 1 else self.P[l] @ X @ self.P[l].T

    def to_fine(self, l, X):
        """I_l^1: interpolate a level-l vector up to level 1."""
        for k in range(l - 1, -1, -1):
            X = self.interpolate(k, X)
        return X

    def coarse(self, Y):
        sh = Y.shape
        return (Y.reshape(sh[0], -1) @ self.Ainv.T).reshape(sh)

    def level_filter(self, l, Hv):
        """F'_l(h) = Re(IDFT(m'_l (.) DFT(h))) (2D P:415)."""
        m = self.mask_level[l]
        if self.dim == 1:
            return torch.fft.ifft(m * torch.fft.fft(Hv, dim=-1), dim=-1).real
        return torch.fft.ifft2(m * torch.fft.fft2(Hv, dim=(-2, -1)), dim=(-2, -1)).real

    def fine_loss(self, l, E):
        """|| m_l (.) DFT_1(E) ||^2 per sample / n_1 (Parseval-normalised), l 0-based."""
        m = self.mask_fine[l]
        if self.dim == 1:
            Z = torch.fft.fft(E, dim=-1)
            return ((m * Z.abs()) ** 2).sum(-1) / E.shape[-1]
        Z = torch.fft.fft2(E, dim=(-2, -1))
        return ((m * Z.abs()) ** 2).sum((-2, -1)) / (E.shape[-1] * E.shape[-2])


def rhs_norm(X):
    return X.reshape(X.shape[0], -1).norm(dim=1)


# ------------------------------------------------------------------------------------------
# CNN smoother (reading R7), parameters in PyTorch state_dict order
# ------------------------------------------------------------------------------------------
class CNN(torch.nn.Module):
    def __init__(self, cfg, flat: np.ndarray, out_scale: float = 1.0, device="cpu", dtype=torch.float32):
        super().__init__()
        self.dim = cfg.dim
        self.out_scale = out_scale
        layers = ni.unflatten_params(cfg, np.asarray(flat, np.float64))
        self.w = torch.nn.ParameterList()
        self.b = torch.nn.ParameterList()
        for i, (W, b) in enumerate(layers):
            if i == len(layers) - 1:          # trained without the 1/alpha gain (folded on export)
                W, b = W / out_scale, b / out_scale
            self.w.append(torch.nn.Parameter(torch.tensor(W, dtype=dtype, device=device)))
            self.b.append(torch.nn.Parameter(torch.tensor(b, dtype=dtype, device=device)))

    def forward(self, u):
        z = u[:, None]
        conv = F.conv1d if self.dim == 1 else F.conv2d
        for i in range(len(self.w)):
            z = conv(z, self.w[i], self.b[i], padding=self.w[i].shape[-1] // 2)
            if i + 1 < len(self.w):
                z = F.relu(z)
        return z[:, 0] * self.out_scale

    def export(self) -> np.ndarray:
        """Flat fp32 vector of the equivalent plain CNN (1/alpha folded into the last layer)."""
        layers = []
        for i in range(len(self.w)):
            W = self.w[i].detach().double().cpu().numpy()
            b = self.b[i].detach().double().cpu().numpy()
            if i == len(self.w) - 1:
                W, b = W * self.out_scale, b * self.out_scale
            layers.append((W, b))
        return ni.flatten_params(layers)


class FNO(torch.nn.Module):
    """The paper's FNO smoother (Appendix A, Table 6; readings R23/R24) for level n:
    lift 1 -> c, L Fourier layers GELU(irfft(R . rfft(Z)_k) + W * Z + B), proj c -> 1.  Same flat
    parameter layout as the library's nmg_load_fno_weights (nmg_inputs.fno_param_shapes)."""

    def __init__(self, dim, n, flat, out_scale: float = 1.0, device="cpu", dtype=torch.float32, width=None):
        super().__init__()
        self.dim, self.n, self.out_scale = dim, n, out_scale
        self.arch = ni.fno_arch(dim, n, width)
        c, L, k, ks = self.arch
        P = ni.fno_unflatten(dim, c, L, k, ks, np.asarray(flat, np.float64))
        t = lambda a: torch.nn.Parameter(torch.tensor(a, dtype=dtype, device=device))   # noqa: E731
        self.lift_w, self.lift_b = t(P["lift_w"]), t(P["lift_b"])
        self.spec = torch.nn.ParameterList([t(P[f"spec{i}"]) for i in range(L)])
        self.conv = torch.nn.ParameterList([t(P[f"conv{i}"]) for i in range(L)])
        self.bias = torch.nn.ParameterList([t(P[f"bias{i}"]) for i in range(L)])
        self.proj_w = t(P["proj_w"] / out_scale)
        self.proj_b = t(P["proj_b"] / out_scale)

    def forward(self, u):
        c, L, k, ks = self.arch
        n = self.n
        z = F.linear(u[..., None], self.lift_w, self.lift_b).movedim(-1, 1)      # [B][c][...]
        for i in range(L):
            R = torch.complex(self.spec[i][..., 0], self.spec[i][..., 1])
            if self.dim == 1:
                Z = torch.fft.rfft(z, dim=-1)[..., :k]
                Yp = torch.zeros(z.shape[0], c, n // 2 + 1, dtype=Z.dtype, device=z.device)
                Yp[..., :k] = torch.einsum("bcm,mco->bom", Z, R)
                sp = torch.fft.irfft(Yp, n=n, dim=-1)
                w = F.conv1d(z, self.conv[i], self.bias[i], padding=ks // 2)
            else:
                Z = torch.fft.rfft2(z)
                Yp = torch.zeros(z.shape[0], c, n, n // 2 + 1, dtype=Z.dtype, device=z.device)
                Yp[:, :, :k, :k] = torch.einsum("bcjm,jmco->bojm", Z[:, :, :k, :k], R[:k])
                Yp[:, :, n - k:, :k] = torch.einsum("bcjm,jmco->bojm", Z[:, :, n - k:, :k], R[k:])
                sp = torch.fft.irfft2(Yp, s=(n, n))
                w = F.conv2d(z, self.conv[i], self.bias[i], padding=ks // 2)
            z = F.gelu(sp + w)
        return F.linear(z.movedim(1, -1), self.proj_w, self.proj_b)[..., 0] * self.out_scale

    def export(self) -> np.ndarray:
        parts = [self.lift_w, self.lift_b]
        for i in range(len(self.spec)):
            parts += [self.spec[i], self.conv[i], self.bias[i]]
        out = [p.detach().double().cpu().numpy().ravel() for p in parts]
        out += [(self.proj_w.detach().double().cpu().numpy() * self.out_scale).ravel(),
                (self.proj_b.detach().double().cpu().numpy() * self.out_scale).ravel()]
        return np.concatenate(out).astype(np.float32)


def make_nets(cfg, weights, arch, out_scale=1.0, device="cpu", dtype=torch.float32):
    if arch == "fno":
        return [FNO(cfg.dim, cfg.n >> l, w, out_scale, device, dtype) for l, w in enumerate(weights)]
    return [CNN(cfg, w, out_scale, device, dtype) for w in weights]


def smooth(lv: TorchLevels, nets, l, x, y):
    """One smoothing step (Alg 3): b = y - A x, h = N(b/||b||)||b||, x + F'(h)."""
    b = y - lv.apply(l, x) if x is not None else y
    s = rhs_norm(b)
    shape = (-1,) + (1,) * (b.dim() - 1)
    safe = torch.where(s > 0, s, torch.ones_like(s)).reshape(shape)
    h = nets[l](b / safe) * safe
    h = torch.where(s.reshape(shape) > 0, h, torch.zeros_like(h))
    hf = lv.level_filter(l, h)
    return hf if x is None else x + hf


@torch.no_grad()
def nmgf0(lv: TorchLevels, nets, y, nu1=1, nu2=1, l=0):
    """NMGF(0, y) at level l with nu1 / nu2 smoothing steps (Alg 3/4 + reading R9)."""
    if l == lv.L - 1:
        return lv.coarse(y)
    x = None
    for _ in range(nu1):
        x = smooth(lv, nets, l, x, y)
    if x is None:
        x = torch.zeros_like(y)
    yc = lv.restrict(l, y - lv.apply(l, x))
    x = x + lv.interpolate(l, nmgf0(lv, nets, yc, nu1, nu2, l + 1))
    for _ in range(nu2):
        x = smooth(lv, nets, l, x, y)
    return x


def level_losses(lv: TorchLevels, nets, x_true, y):
    """[L_l for l = 1 .. L-1] (eq. loss_2_modified / loss_3) on one batch; nu1 = 1, nu2 = 0."""
    losses = []
    acc = torch.zeros_like(x_true)              # sum_{k<l} I_k^1 F'_k(h_k), detached
    yl = y
    for l in range(lv.L - 1):
        b = yl.detach()
        s = rhs_norm(b)
        shape = (-1,) + (1,) * (b.dim() - 1)
        safe = torch.where(s > 0, s, torch.ones_like(s)).reshape(shape)
        h = nets[l](b / safe) * safe
        e = x_true - acc - lv.to_fine(l, h)
        losses.append(lv.fine_loss(l, e).mean())
        hf = lv.level_filter(l, h).detach()
        acc = acc + lv.to_fine(l, hf)
        yl = lv.restrict(l, b - lv.apply(l, hf))
    return losses


# ------------------------------------------------------------------------------------------
# DataGeneration (Alg 5) with the rollout through the library or the transcription
# ------------------------------------------------------------------------------------------
class NmgRollout:
    """x <- NMGF(0, y) through the C ABI (nmg_vcycle from x = 0: x + NMGF(0, y - A x))."""

    def __init__(self, cfg, factors, alpha, nbs):
        import paper_2603_01064_b200 as nmg
        self.cfg = cfg
        self.h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, alpha, factors, nu1=cfg.nu1, nu2=cfg.nu2,
                               max_rhs=nbs)

    def load(self, nets):
        for l, net in enumerate(nets):
            if isinstance(net, FNO):
                self.h.load_fno_weights(l + 1, net.arch, net.export())
            else:
                self.h.load_weights(l + 1, ni.cnn_arch(self.cfg), net.export())

    def __call__(self, y):
        yd = y.to(torch.float64).contiguous()
        x = torch.zeros_like(yd)
        self.h.vcycle(yd, x)
        torch.cuda.synchronize()
        return x.to(y.dtype)


def data_generation(lv: TorchLevels, nets, nbs: int, K: int, rng: np.random.Generator, rollout=None,
                    nu1: int = 1, nu2: int = 1):
    shape = (nbs,) + ((lv.ns[0],) if lv.dim == 1 else (lv.ns[0], lv.ns[0]))
    x = torch.tensor(rng.standard_normal(shape), dtype=lv.dt, device=lv.dev)
    y = lv.apply(0, x)
    ks = rng.integers(1, K + 1, size=nbs)
    shape_b = (-1,) + (1,) * (x.dim() - 1)
    for j in range(1, K + 1):
        live = torch.tensor(ks >= j, device=lv.dev)
        if not bool(live.any()):
            break
        with torch.no_grad():
            c = rollout(y) if rollout is not None else nmgf0(lv, nets, y, nu1, nu2)
        xn = x - c
        # a cycle of a still-untrained smoother may diverge: such a sample keeps its last finite
        # error (and stops rolling); the rest are rescaled to unit norm after every step (the
        # cycle is positively homogeneous, pin P10), so no rollout overflows
        nrm = rhs_norm(xn)
        ok = torch.isfinite(nrm) & (nrm > 0) & live
        ks = np.where(ok.cpu().numpy(), ks, 0)
        xn = xn / torch.where(ok, nrm, torch.ones_like(nrm)).reshape(shape_b)
        x = torch.where(ok.reshape(shape_b), xn, x)
        y = lv.apply(0, x)
    nx = rhs_norm(x).reshape((-1,) + (1,) * (x.dim() - 1))
    nx = torch.where(nx > 0, nx, torch.ones_like(nx))
    return x / nx, y / nx


# ------------------------------------------------------------------------------------------
def train(cfg, alpha: float, init: List[np.ndarray], epochs: int, nbs: int = 20, K: int = 10, lr: float = 1e-3,
          device="cpu", seed: int = 0, rollout: str = "torch", log_every: int = 100, verbose=True, arch="cnn"):
    factors = ni.operator_factors(cfg)
    lv = TorchLevels(cfg, factors, alpha, device)
    nets = make_nets(cfg, init, arch, out_scale=1.0 / alpha, device=device)
    opts = [torch.optim.Adam(n.parameters(), lr=lr) for n in nets]
    # linear warm-up over the first 5 % of the epochs (a curriculum stage starts from the previous
    # alpha's smoother under a 10x larger output gain), then cosine decay to 2 % of lr
    warm = max(1, epochs // 20)
    sched_fn = lambda e: (e + 1) / warm if e < warm else 0.02 + 0.49 * (1 + math.cos(math.pi * (e - warm) / max(1, epochs - warm)))   # noqa: E731
    scheds = [torch.optim.lr_scheduler.LambdaLR(o, sched_fn) for o in opts]
    ro = NmgRollout(cfg, factors, alpha, nbs) if rollout == "nmg" else None
    rng = np.random.default_rng(seed)
    hist = []
    t0 = time.time()
    for ep in range(epochs):
        if ro is not None:
            ro.load(nets)
        x, y = data_generation(lv, nets, nbs, K, rng, ro, cfg.nu1, cfg.nu2)
        losses = level_losses(lv, nets, x, y)
        for o in opts:
            o.zero_grad(set_to_none=True)
        total = sum(losses)
        if bool(torch.isfinite(total)):          # a non-finite batch is skipped, not learned from
            total.backward()
            for net in nets:
                torch.nn.utils.clip_grad_norm_(net.parameters(), 10.0)
            for o in opts:
                o.step()
        for sch in scheds:
            sch.step()
        hist.append([float(v.detach()) for v in losses])
        if verbose and (ep % log_every == 0 or ep == epochs - 1):
            print(f"  alpha {alpha:g} epoch {ep:5d}  losses " + " ".join(f"{v:.3e}" for v in hist[-1])
                  + f"  ({time.time() - t0:.0f} s)", flush=True)
    return [n.export() for n in nets], np.array(hist)


@torch.no_grad()
def eval_solve(cfg, alpha, weights, nrhs=16, max_cycles=100, device="cpu", tol=1e-6, arch="cnn"):
    """Relative-residual histories of the trained cycle (transcription, fp64) on the problem's
    own seeded right-hand sides: a quick convergence check (the parity check is the oracle's)."""
    factors = ni.operator_factors(cfg)
    lv = TorchLevels(cfg, factors, alpha, device, dtype=torch.float64)
    nets = make_nets(cfg, weights, arch, device=device, dtype=torch.float64)
    y, _ = ni.make_rhs(cfg, factors, alpha, nrhs=nrhs)
    y = torch.tensor(y, dtype=torch.float64, device=device)
    x = torch.zeros_like(y)
    ny = rhs_norm(y)
    hist = [torch.ones(nrhs, dtype=torch.float64)]
    for _ in range(max_cycles):
        r = y - lv.apply(0, x)
        x = x + nmgf0(lv, nets, r, cfg.nu1, cfg.nu2)
        rr = rhs_norm(y - lv.apply(0, x)) / ny
        hist.append(rr.cpu())
        if bool((rr <= tol).all()) or not bool(torch.isfinite(rr).all()):
            break
    return torch.stack(hist, 1).numpy()


def save(cfg, alpha, weights, hist, extra=None, out_dir=OUT_DIR, arch="cnn"):
    os.makedirs(out_dir, exist_ok=True)
    tag = "" if arch == "cnn" else "_fno"
    p = os.path.join(out_dir, f"W_train{tag}_{cfg.name}_a{alpha:g}.npz")
    w = np.stack(weights) if arch == "cnn" else np.array(weights, dtype=object)
    np.savez_compressed(p, weights=w, loss_history=hist, alpha=alpha, config=cfg.name, **(extra or {}))
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--alphas", type=float, nargs="+", default=None, help="curriculum, large -> small (P:477)")
    ap.add_argument("--epochs", type=int, default=1500)
    ap.add_argument("--nbs", type=int, default=20)
    ap.add_argument("--K", type=int, default=10)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--rollout", choices=["nmg", "torch"], default=None)
    ap.add_argument("--init", choices=["seed", "lin", "trained"], default="seed",
                    help="trained: start from nmg_inputs/trained at --init-alpha")
    ap.add_argument("--init-alpha", type=float, default=None)
    ap.add_argument("--n", type=int, default=None, help="override the grid size (quick runs)")
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--out", default=OUT_DIR)
    ap.add_argument("--arch", choices=["cnn", "fno"], default="cnn", help="fno: the paper's smoother (Table 6)")
    args = ap.parse_args()
    cfg = ni.CONFIGS[args.config]
    if args.n:
        cfg = cfg.replace(n=args.n, levels=args.levels or cfg.levels)
    alphas = args.alphas or ni.ALPHAS[args.config]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    rollout = args.rollout or ("nmg" if dev == "cuda" else "torch")
    if args.arch == "fno":
        w = ni.fno_weights_seed(cfg)
    elif args.init == "trained":
        w = ni.weights_trained(cfg.replace(alpha=args.init_alpha))
        assert w is not None, "no trained weights at --init-alpha"
    else:
        w = ni.weights_seed(cfg) if args.init == "seed" else ni.weights_lin(cfg, alpha=alphas[0])
    for a in sorted(alphas, reverse=True):
        c = cfg.replace(alpha=a)
        t0 = time.time()
        w, hist = train(c, a, w, args.epochs, args.nbs, args.K, args.lr, dev, rollout=rollout, arch=args.arch)
        h = eval_solve(c, a, w, device=dev, arch=args.arch)
        last = h[:, -1]
        print(f"alpha {a:g}: trained in {time.time() - t0:.0f} s; eval {h.shape[1] - 1} cycles, "
              f"max final relres {np.nanmax(last):.3e}", flush=True)
        print("saved", save(c, a, w, hist, {"eval_history": h}, args.out, args.arch), flush=True)


if __name__ == "__main__":
    main()
