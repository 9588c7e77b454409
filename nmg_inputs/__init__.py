"""Seeded synthetic inputs for the batched NMGF solve (arxiv 2603.01064).

This module is shared by the oracle (``oracle/``) and the CUDA path
(``paper_2603_01064_b200``).  It holds only PROBLEM DATA -- the
discretised kernels that define A, the right-hand sides and the smoother
weights -- and none of the method's arithmetic (no transfers, no Galerkin
chain, no masks/filters, no CNN evaluation, no cycle).  Every random number
the method consumes is drawn here and passed in as an input.

Recipes (readings R2, R8, R15, R16, R17 in DESIGN.md):

* 1D kernel (BASELINE.json configs[0]):
  ``t_i = (i+1/2)/n``, ``K_ij = h exp(-(t_i-t_j)^2/(2 sigma^2)) / (sigma sqrt(2 pi))``,
  ``h = 1/n``, no wrap (Toeplitz, section 2.1).
  System ``A = K^T K + alpha I`` (BASELINE configs[0]; the paper's own form
  ``alpha I + K`` (eq. eq:1d_linear_system) is ``paper_form=True``).
* 2D (configs[2], [3]): ``K = K1 (x) K1`` so ``G = K^T K = M (x) M`` with
  ``M = K1^T K1``; A = G + alpha I, applied as ``C X B^T`` on the column-major
  matrix X (Vec convention).
* 2D config 4: kernel ``exp(-|d|^2/(2 sigma^2)) (1 + 0.3 cos(2 pi d1))`` is a
  product of a factor in d1 and one in d2, so ``K = K_(2) (x) K_(1)`` with the
  cos factor on axis 1 (i1, the fastest axis) -- reading R17.
* RHS 1D (R15): per RHS, f ~ U{1..fmax} x5, a ~ N(0,1) x5,
  ``x*(t) = sum a_j sin(2 pi f_j t)``, noise N(0, std 1e-3), ``y = A x* + noise``;
  ``numpy.random.default_rng(1)``.
* RHS 2D (R16): m ~ U{10..30} Gaussian blobs, centres U[0,1]^2, widths
  U(0.01, 0.1), amplitudes N(0,1), plus N(0, std 1e-3) noise; ``y = A x* + noise``.
* W_seed (R8): He-uniform ``U(+-sqrt(6/fan_in))`` weights, bias
  ``U(+-1/sqrt(fan_in))``, ``default_rng(0)``, drawn level 1..L-1, layer by
  layer, weight then bias, C order; stored fp32 in PyTorch state_dict order.
* W_lin / W_zero: deterministic CNN weights that make the smoother exactly
  linear (ReLU(z) - ReLU(-z) = z) or identically zero.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

# --------------------------------------------------------------------------
# Configurations (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dim: int            # 1 or 2
    n: int              # points per axis on the finest grid
    sigma: float
    alpha: float
    levels: int         # L (level L is the exact coarse solve)
    nrhs: int
    channels: int       # CNN width
    n_layers: int       # CNN depth
    ksize: int          # CNN kernel width (per axis)
    fmax: int = 40      # 1D sinusoid frequency range 1..fmax
    kernel: str = "gauss"   # "gauss" | "gauss_cos" (config 4)
    nu1: int = 1
    nu2: int = 1
    cycles: int = 10

    @property
    def N(self) -> int:
        return self.n if self.dim == 1 else self.n * self.n

    def level_sizes(self) -> List[int]:
        return [self.n >> l for l in range(self.levels)]

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    0: Config("cfg0_1d_tiny", 1, 256, 0.05, 1e-3, 3, 8, 16, 3, 5, fmax=40),
    1: Config("cfg1_1d_mid", 1, 4096, 0.02, 1e-3, 6, 1024, 16, 3, 5, fmax=500),
    2: Config("cfg2_2d", 2, 256, 0.03, 1e-3, 5, 256, 32, 4, 3),
    3: Config("cfg3_2d_large", 2, 512, 0.02, 1e-3, 6, 2048, 48, 4, 3),
    4: Config("cfg4_2d_huge", 2, 1024, 0.02, 1e-4, 7, 32, 32, 4, 3, kernel="gauss_cos"),
}
# alpha sweeps named by BASELINE.json
ALPHAS = {0: [1e-3], 1: [1e-2, 1e-3, 1e-4], 2: [1e-3], 3: [1e-3, 1e-4], 4: [1e-4]}


# --------------------------------------------------------------------------
# Operators (problem definition, not the method)
# --------------------------------------------------------------------------

def grid_points(n: int) -> np.ndarray:
    """Cell centres t_i = (i + 1/2)/n (BASELINE configs[0])."""
    return (np.arange(n, dtype=np.float64) + 0.5) / n


def gaussian_kernel_1d(n: int, sigma: float, cos_mod: float = 0.0) -> np.ndarray:
    """K_ij = h exp(-(t_i-t_j)^2/(2 s^2)) (1 + cos_mod cos(2 pi (t_i-t_j))) / (s sqrt(2 pi)).

    cos_mod = 0 is the BASELINE configs[0] formula; cos_mod = 0.3 is the
    axis-1 factor of configs[4] (reading R17).
    """
    t = grid_points(n)
    d = t[:, None] - t[None, :]
    h = 1.0 / n
    K = h * np.exp(-d * d / (2.0 * sigma * sigma)) / (sigma * math.sqrt(2.0 * math.pi))
    if cos_mod:
        K = K * (1.0 + cos_mod * np.cos(2.0 * math.pi * d))
    return K


def _sym_gram(K: np.ndarray) -> np.ndarray:
    """K^T K, made bitwise symmetric (PAPER form is SPD; see pin P1)."""
    G = K.T @ K
    return 0.5 * (G + G.T)


def operator_factors(cfg: Config, paper_form: bool = False) -> Tuple[np.ndarray, ...]:
    """Structured G of A = G + alpha I.

    1D: returns (G,) with G dense n x n (row-major, symmetric).
    2D: returns (B, C) with G = B (x) C, i.e. G Vec(X) = Vec(C X B^T);
        C acts along i1 (fastest axis), B along i2.
    paper_form=True gives G = K (1D) / K (x) K (2D).
    """
    if cfg.dim == 1:
        K = gaussian_kernel_1d(cfg.n, cfg.sigma)
        return ((K.copy() if paper_form else _sym_gram(K)),)
    if cfg.kernel == "gauss":
        K1 = gaussian_kernel_1d(cfg.n, cfg.sigma)
        M = K1.copy() if paper_form else _sym_gram(K1)
        return (M, M.copy())
    if cfg.kernel == "gauss_cos":
        K_a = gaussian_kernel_1d(cfg.n, cfg.sigma, cos_mod=0.3)   # axis 1 (i1)
        K_b = gaussian_kernel_1d(cfg.n, cfg.sigma)                # axis 2 (i2)
        if paper_form:
            return (K_b, K_a)
        return (_sym_gram(K_b), _sym_gram(K_a))
    raise ValueError(cfg.kernel)


def anisotropic_factors(cfg: Config, alpha: float) -> Tuple[np.ndarray]:
    """The paper's anisotropic 1D system A = alpha D + K with D = diag(a(t_i)),
    a(z) = 1 + 0.5 sin(2 pi z), as the G of A = G + alpha I:
    G = K + alpha (D - I) (dense, symmetric).  Problem data only."""
    assert cfg.dim == 1
    K = gaussian_kernel_1d(cfg.n, cfg.sigma)
    a = 1.0 + 0.5 * np.sin(2.0 * math.pi * grid_points(cfg.n))
    G = K + alpha * np.diag(a - 1.0)
    return (0.5 * (G + G.T),)


def truncated_kernel_2d_cfg4(n: int, sigma: float, tol: float = 1e-12):
    """Direct (non-Kronecker) config-4 stencil, truncated where the unnormalised
    value exp(-|d|^2/(2 s^2)) (1 + 0.3 cos(2 pi d1)) < tol (reading R2/R17).
    Returns (offsets (m,2) int, weights (m,)) with d = offsets / n.
    """
    h = 1.0 / n
    r = int(math.ceil(sigma * math.sqrt(2.0 * math.log(1.3 / tol)) * n)) + 1
    o = np.arange(-r, r + 1)
    d1 = o[:, None] * h
    d2 = o[None, :] * h
    un = np.exp(-(d1 * d1 + d2 * d2) / (2 * sigma * sigma)) * (1.0 + 0.3 * np.cos(2 * math.pi * d1))
    keep = un >= tol
    w = h * h * un / (2.0 * math.pi * sigma * sigma)
    i1, i2 = np.nonzero(keep)
    return np.stack([o[i1], o[i2]], axis=1), w[i1, i2]


# --------------------------------------------------------------------------
# Right-hand sides
# --------------------------------------------------------------------------

def apply_A_problem(cfg: Config, factors, alpha: float, X: np.ndarray) -> np.ndarray:
    """y = A x* used ONLY to manufacture right-hand sides (problem data).

    X layout: 1D [b][i]; 2D [b][i2][i1] (column-major per RHS).
    """
    if cfg.dim == 1:
        (G,) = factors
        return X @ G.T + alpha * X
    B, C = factors
    # Vec(C X B^T) with arr[b] = X_b^T  ->  B @ arr[b] @ C^T
    return np.matmul(np.matmul(B, X), C.T) + alpha * X


def rhs_1d(cfg: Config, factors, alpha: float, nrhs: Optional[int] = None,
           seed: int = 1, start: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(y, x*) for configs[0]/[1]; reading R15.  RHS index b uses draws in order
    b = 0, 1, ...; ``start`` skips the first ``start`` RHS (same stream)."""
    nrhs = cfg.nrhs if nrhs is None else nrhs
    rng = np.random.default_rng(seed)
    t = grid_points(cfg.n)
    xs = np.empty((nrhs, cfg.n))
    noise = np.empty((nrhs, cfg.n))
    for b in range(start + nrhs):
        f = rng.integers(1, cfg.fmax + 1, size=5)
        a = rng.standard_normal(5)
        nz = rng.normal(0.0, 1e-3, size=cfg.n)
        if b >= start:
            xs[b - start] = (a[:, None] * np.sin(2.0 * math.pi * f[:, None] * t[None, :])).sum(0)
            noise[b - start] = nz
    y = apply_A_problem(cfg, factors, alpha, xs) + noise
    return y, xs


def rhs_2d(cfg: Config, factors, alpha: float, nrhs: Optional[int] = None,
           seed: int = 1, start: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(y, x*) for configs[2..4]; reading R16.  Layout [b][i2][i1]."""
    nrhs = cfg.nrhs if nrhs is None else nrhs
    rng = np.random.default_rng(seed)
    t = grid_points(cfg.n)
    xs = np.zeros((nrhs, cfg.n, cfg.n))
    noise = np.empty((nrhs, cfg.n, cfg.n))
    for b in range(start + nrhs):
        m = int(rng.integers(10, 31))
        c = rng.uniform(0.0, 1.0, size=(m, 2))
        w = rng.uniform(0.01, 0.1, size=m)
        a = rng.standard_normal(m)
        nz = rng.normal(0.0, 1e-3, size=(cfg.n, cfg.n))
        if b >= start:
            acc = np.zeros((cfg.n, cfg.n))
            for j in range(m):
                g1 = np.exp(-(t - c[j, 0]) ** 2 / (2 * w[j] ** 2))   # along i1
                g2 = np.exp(-(t - c[j, 1]) ** 2 / (2 * w[j] ** 2))   # along i2
                acc += a[j] * g2[:, None] * g1[None, :]
            xs[b - start] = acc
            noise[b - start] = nz
    y = apply_A_problem(cfg, factors, alpha, xs) + noise
    return y, xs


def make_rhs(cfg: Config, factors, alpha: float, nrhs=None, seed: int = 1, start: int = 0):
    if cfg.dim == 1:
        return rhs_1d(cfg, factors, alpha, nrhs, seed, start)
    return rhs_2d(cfg, factors, alpha, nrhs, seed, start)


# --------------------------------------------------------------------------
# Smoother weights (CNN, reading R7), PyTorch state_dict order
# --------------------------------------------------------------------------

def layer_shapes(cfg: Config) -> List[Tuple[Tuple[int, ...], Tuple[int]]]:
    """[(weight_shape, bias_shape)] per layer: 1 -> C -> ... -> C -> 1."""
    C, k, L = cfg.channels, cfg.ksize, cfg.n_layers
    chans = [1] + [C] * (L - 1) + [1]
    out = []
    for i in range(L):
        ks = (k,) if cfg.dim == 1 else (k, k)
        out.append(((chans[i + 1], chans[i]) + ks, (chans[i + 1],)))
    return out


def n_params(cfg: Config) -> int:
    return sum(int(np.prod(w)) + int(np.prod(b)) for w, b in layer_shapes(cfg))


def flatten_params(layers: Sequence[Tuple[np.ndarray, np.ndarray]]) -> np.ndarray:
    return np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in layers]).astype(np.float32)


def unflatten_params(cfg: Config, flat: np.ndarray):
    layers, o = [], 0
    for ws, bs in layer_shapes(cfg):
        nw, nb = int(np.prod(ws)), int(np.prod(bs))
        layers.append((flat[o:o + nw].reshape(ws), flat[o + nw:o + nw + nb].reshape(bs)))
        o += nw + nb
    assert o == flat.size
    return layers


def weights_seed(cfg: Config, seed: int = 0) -> List[np.ndarray]:
    """W_seed: one flat fp32 parameter vector per smoothed level 1..L-1 (R8)."""
    rng = np.random.default_rng(seed)
    out = []
    for _lvl in range(1, cfg.levels):
        layers = []
        for ws, bs in layer_shapes(cfg):
            fan_in = int(np.prod(ws[1:]))
            wb = math.sqrt(6.0 / fan_in)
            w = rng.uniform(-wb, wb, size=ws)
            bb = 1.0 / math.sqrt(fan_in)
            b = rng.uniform(-bb, bb, size=bs)
            layers.append((w, b))
        out.append(flatten_params(layers))
    return out


def weights_zero(cfg: Config) -> List[np.ndarray]:
    return [np.zeros(n_params(cfg), np.float32) for _ in range(1, cfg.levels)]


def _delta(cfg: Config) -> np.ndarray:
    k = cfg.ksize
    if cfg.dim == 1:
        d = np.zeros(k)
        d[k // 2] = 1.0
    else:
        d = np.zeros((k, k))
        d[k // 2, k // 2] = 1.0
    return d


def default_g1(cfg: Config) -> np.ndarray:
    """High-pass first filter of W_lin: [-1/4, 1/2, -1/4] (1D) or the 5-point
    (4 delta - N - S - E - W)/8 (2D), centred in the k-wide kernel."""
    k = cfg.ksize
    c = k // 2
    if cfg.dim == 1:
        g = np.zeros(k)
        g[c - 1], g[c], g[c + 1] = -0.25, 0.5, -0.25
    else:
        g = np.zeros((k, k))
        g[c, c] = 0.5
        g[c - 1, c] = g[c + 1, c] = g[c, c - 1] = g[c, c + 1] = -0.125
    return g


def weights_lin(cfg: Config, scale: Optional[float] = None, g1=None, alpha: Optional[float] = None):
    """W_lin: CNN realising h = scale * (g_last * ... * g1) * b exactly
    (middle filters are deltas).  Uses ReLU(z) - ReLU(-z) = z with two live
    channels; all biases 0.  scale defaults to 1/alpha.
    """
    alpha = cfg.alpha if alpha is None else alpha
    scale = (1.0 / alpha) if scale is None else scale
    g1 = default_g1(cfg) if g1 is None else np.asarray(g1, dtype=np.float64)
    d = _delta(cfg)
    shapes = layer_shapes(cfg)
    layers = []
    for i, (ws, bs) in enumerate(shapes):
        w = np.zeros(ws)
        b = np.zeros(bs)
        if i == 0:
            w[0, 0], w[1, 0] = g1, -g1
        elif i == len(shapes) - 1:
            w[0, 0], w[0, 1] = scale * d, -scale * d
        else:
            w[0, 0], w[0, 1], w[1, 0], w[1, 1] = d, -d, -d, d
        layers.append((w, b))
    return [flatten_params(layers) for _ in range(1, cfg.levels)]


def cnn_arch(cfg: Config) -> Tuple[int, int, int]:
    return (cfg.n_layers, cfg.channels, cfg.ksize)


# --------------------------------------------------------------------------
# FNO smoother (Appendix A, Table 6)
# --------------------------------------------------------------------------
# Table 6 (tab:network_structures): per grid h = 1/n the width c, Fourier layers L, retained
# modes k and W-convolution kernel size.  Grids outside the table take the nearest row with
# k capped at n/4 (reading R23 in DESIGN.md).
FNO_TABLE = {
    1: {64: (64, 4, 16, 5), 128: (64, 4, 32, 5), 256: (64, 5, 64, 7), 512: (64, 6, 128, 7), 1024: (64, 6, 128, 7)},
    2: {64: (64, 4, 16, 3), 128: (64, 4, 32, 3), 256: (64, 5, 32, 5), 512: (64, 6, 64, 7), 1024: (64, 6, 64, 7)},
}


def fno_arch(dim: int, n: int, width: Optional[int] = None) -> Tuple[int, int, int, int]:
    """(c, L, k, ksize) for a level with n points per axis (Table 6, nearest row)."""
    rows = FNO_TABLE[dim]
    key = min(rows, key=lambda r: abs(math.log2(r) - math.log2(n)))
    c, L, k, ks = rows[key]
    k = max(1, min(k, n // 4))
    return (width or c, L, k, ks)


def fno_param_shapes(dim: int, c: int, L: int, k: int, ks: int) -> List[Tuple[str, Tuple[int, ...]]]:
    """Flat parameter order (the ABI's, nmg.h nmg_load_fno_weights):
    lift.w [c][1], lift.b [c]; per Fourier layer: spectral R ([k][c_in][c_out][re,im] in 1D,
    [2k][k][c_in][c_out][re,im] in 2D: i2-mode rows 0..k-1 then n-k..n-1, i1-modes 0..k-1),
    conv W [c_out][c_in][ks](x ks), bias [c]; proj.w [1][c], proj.b [1]."""
    spec = (k, c, c, 2) if dim == 1 else (2 * k, k, c, c, 2)
    conv = (c, c, ks) if dim == 1 else (c, c, ks, ks)
    out = [("lift_w", (c, 1)), ("lift_b", (c,))]
    for i in range(L):
        out += [(f"spec{i}", spec), (f"conv{i}", conv), (f"bias{i}", (c,))]
    out += [("proj_w", (1, c)), ("proj_b", (1,))]
    return out


def fno_n_params(dim, c, L, k, ks) -> int:
    return sum(int(np.prod(sh)) for _, sh in fno_param_shapes(dim, c, L, k, ks))


def fno_unflatten(dim, c, L, k, ks, flat: np.ndarray) -> dict:
    out, o = {}, 0
    for name, sh in fno_param_shapes(dim, c, L, k, ks):
        m = int(np.prod(sh))
        out[name] = np.asarray(flat[o:o + m]).reshape(sh)
        o += m
    assert o == flat.size
    return out


def fno_weights_seed(cfg: Config, seed: int = 0, width: Optional[int] = None) -> List[np.ndarray]:
    """W_seed for FNO smoothers, one flat fp32 vector per smoothed level (arch from fno_arch):
    PyTorch-default-style bounds -- lift / proj / conv U(+-1/sqrt(fan_in)) weights and biases,
    spectral weights (1/(c c)) U(0, 1) for the real and imaginary parts (the FNO reference
    initialisation)."""
    rng = np.random.default_rng(seed)
    out = []
    for lvl in range(cfg.levels - 1):
        n = cfg.n >> lvl
        c, L, k, ks = fno_arch(cfg.dim, n, width)
        parts = []
        for name, sh in fno_param_shapes(cfg.dim, c, L, k, ks):
            if name.startswith("spec"):
                parts.append(rng.uniform(0.0, 1.0, size=sh) / (c * c))
            else:
                fan_in = {"lift_w": 1, "lift_b": 1, "proj_w": c, "proj_b": c}.get(name, c * ks ** cfg.dim)
                bd = 1.0 / math.sqrt(fan_in)
                parts.append(rng.uniform(-bd, bd, size=sh))
        out.append(np.concatenate([p.ravel() for p in parts]).astype(np.float32))
    return out


# --------------------------------------------------------------------------
# W_train: smoothers trained by trainer/nmg_train.py (Alg 5, NEXT-1), committed as data
# --------------------------------------------------------------------------
TRAINED_DIR = __import__("os").path.join(__import__("os").path.dirname(__file__), "trained")


def trained_path(cfg: Config) -> str:
    import os
    return os.path.join(TRAINED_DIR, f"W_train_{cfg.name}_a{cfg.alpha:g}.npz")


def weights_trained(cfg: Config) -> Optional[List[np.ndarray]]:
    """W_train for (config, alpha) if the trainer's output is present, else None."""
    import os
    p = trained_path(cfg)
    if not os.path.exists(p):
        return None
    with np.load(p) as z:
        w = z["weights"]
    if w.shape != (cfg.levels - 1, n_params(cfg)):
        return None
    return [np.ascontiguousarray(v, dtype=np.float32) for v in w]
