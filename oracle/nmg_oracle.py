"""Plain, slow fp64 CPU oracle of the batched NMGF solve (arxiv 2603.01064).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything under ``oracle/``.  The product path (``paper_2603_01064_b200``)
never imports this module and this module never imports the product; the
two share only the seeded problem data from ``nmg_inputs``.

Citations: ``P:<line>`` is a line of PAPER.md with the enclosing algorithm /
equation; ``R<k>`` is a reading listed in DESIGN.md (section "Readings").

Structure, in the paper's order:
  * transfers I_l^{l+1} (restriction) / I_{l+1}^l (interpolation)   -- R4
  * Galerkin chain A^{(l+1)} = I_l^{l+1} A^{(l)} I_{l+1}^l            -- Alg 1
  * coarsest exact solve (LU with partial pivoting)                  -- Alg 3, R12
  * masks m'_l, filters F'_l                                         -- P:288-306, R5
  * CNN smoother N_theta_l                                            -- R7
  * smoothing step  b = y - A x*, h = N(b/|b|)|b|, x = x* + F'(h)     -- Alg 3
  * NMGF cycle (Alg 3 P:315-339 / Alg 4, with nu2 post steps, R9)
  * outer iteration x^tau = NMGF(x^{tau-1}, y), stop at relres 1e-6  -- P:312-313

Everything is fp64 (numpy float64).  CNN weights arrive as fp32 values and are
used as fp64 numbers.  Library primitives used as single steps: matrix
products (numpy/BLAS), np.fft (DFT), np.tensordot (channel contraction per tap).

parity unpinned: CNN outputs with ReLU active under W_seed beyond the
library-conv comparison (tests/test_oracle_pins.py::test_cnn_*), and the
absolute W_seed residual levels -- see DESIGN.md "Pins".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

# ==========================================================================
# Transfers (reading R4: cell-centred linear interpolation / full weighting)
# ==========================================================================


def interpolation_matrix(n_c: int) -> np.ndarray:
    """I_{l+1}^l as a dense (2 n_c) x n_c matrix (P:162 names it; R4 defines it).

    Fine cell i sits between coarse cells; its nearest coarse cell is i>>1
    (weight 3/4) and its second nearest is (i>>1)+1 for odd i, (i>>1)-1 for
    even i (weight 1/4), clamped to the grid so the two end cells copy.
    """
    n_f = 2 * n_c
    P = np.zeros((n_f, n_c))
    for i in range(n_f):
        j = i >> 1
        k = j + 1 if (i & 1) else j - 1
        k = min(max(k, 0), n_c - 1)
        P[i, j] += 0.75
        P[i, k] += 0.25
    return P


def restriction_matrix(n_f: int) -> np.ndarray:
    """I_l^{l+1} as a dense (n_f/2) x n_f matrix (R4 full weighting).

    Interior: r[j] = (f[2j-1] + 3 f[2j] + 3 f[2j+1] + f[2j+2]) / 8;
    ends: r[0] = (4 f[0] + 3 f[1] + f[2]) / 8,
          r[n_c-1] = (f[n_f-3] + 3 f[n_f-2] + 4 f[n_f-1]) / 8.
    (Written out independently of interpolation_matrix; the test pins
    R = P^T / 2.)
    """
    n_c = n_f // 2
    R = np.zeros((n_c, n_f))
    for j in range(n_c):
        for i, w in ((2 * j - 1, 1.0), (2 * j, 3.0), (2 * j + 1, 3.0), (2 * j + 2, 1.0)):
            i = min(max(i, 0), n_f - 1)   # the clamped end tap folds into the end cell
            R[j, i] += w / 8.0
    return R


# ==========================================================================
# Hierarchy
# ==========================================================================

@dataclass
class Hierarchy:
    dim: int
    alpha: float
    levels: int
    n: List[int]                       # points per axis per level (level 1 first)
    A: List[np.ndarray] = field(default_factory=list)   # 1D: dense A^{(l)}
    Bf: List[np.ndarray] = field(default_factory=list)  # 2D: A^{(l)} = B_l (x) C_l + alpha Q_l (x) Q_l
    Cf: List[np.ndarray] = field(default_factory=list)
    Q: List[np.ndarray] = field(default_factory=list)
    P: List[np.ndarray] = field(default_factory=list)   # P[l] : level l+1 -> level l (index l = 0..L-2)
    R: List[np.ndarray] = field(default_factory=list)
    A_coarse: Optional[np.ndarray] = None                # dense A^{(L)} (2D: N_L x N_L)
    lu: Optional[Tuple[np.ndarray, np.ndarray]] = None
    masks: List[np.ndarray] = field(default_factory=list)
    weights: List[Optional[list]] = field(default_factory=list)   # per smoothed level: [(W, b)]
    nu1: int = 1
    nu2: int = 1
    level_filter: bool = True


def build_hierarchy(dim: int, factors: Sequence[np.ndarray], alpha: float, levels: int,
                    nu1: int = 1, nu2: int = 1, level_filter: bool = True) -> Hierarchy:
    """Galerkin chain A^{(l+1)} = I_l^{l+1} A^{(l)} I_{l+1}^l (Alg 1, used
    unchanged by Alg 3 P:333 and Alg 4), masks m'_l, coarse LU."""
    if dim == 1:
        (G,) = factors
        n = G.shape[0]
    else:
        Bf, Cf = factors
        n = Bf.shape[0]
    ns = [n >> l for l in range(levels)]
    H = Hierarchy(dim=dim, alpha=alpha, levels=levels, n=ns, nu1=nu1, nu2=nu2,
                  level_filter=level_filter)
    for l in range(levels - 1):
        H.P.append(interpolation_matrix(ns[l + 1]))
        H.R.append(restriction_matrix(ns[l]))
    if dim == 1:
        A = np.array(G, dtype=np.float64) + alpha * np.eye(n)
        H.A.append(A)
        for l in range(levels - 1):
            A = H.R[l] @ A @ H.P[l]
            H.A.append(A)
        H.A_coarse = H.A[-1]
    else:
        # 2D: hat I = I (x) I on Vec, so hat R (B (x) C + alpha I (x) I) hat P
        #   = (R B P) (x) (R C P) + alpha (R P) (x) (R P)    (Kronecker mixed product)
        B_, C_, Q_ = np.array(Bf, np.float64), np.array(Cf, np.float64), np.eye(n)
        H.Bf.append(B_); H.Cf.append(C_); H.Q.append(Q_)
        for l in range(levels - 1):
            B_ = H.R[l] @ B_ @ H.P[l]
            C_ = H.R[l] @ C_ @ H.P[l]
            Q_ = H.R[l] @ Q_ @ H.P[l]
            H.Bf.append(B_); H.Cf.append(C_); H.Q.append(Q_)
        # dense coarsest operator on Vec (column-major: index i1 + n i2)
        H.A_coarse = np.kron(H.Bf[-1], H.Cf[-1]) + alpha * np.kron(H.Q[-1], H.Q[-1])
    H.lu = lu_factor(H.A_coarse)
    for l in range(levels - 1):
        H.masks.append(level_mask(ns[l], dim))
    H.weights = [None] * (levels - 1)
    return H


def load_weights(H: Hierarchy, level: int, layers) -> None:
    """Smoother parameters theta_l for level l (1-based, l < L): a CNN as layers = [(W, b)],
    or an FNO as the dict of fno_params()."""
    if isinstance(layers, dict):
        H.weights[level - 1] = layers
        return
    H.weights[level - 1] = [(np.asarray(w, np.float64), np.asarray(b, np.float64)) for w, b in layers]


def apply_A(H: Hierarchy, l: int, X: np.ndarray) -> np.ndarray:
    """A^{(l)} x for a batch; l is 0-based here.  1D X: [b][i]; 2D X: [b][i2][i1].

    2D: Mat(hat A Vec(X)) = C X B^T + alpha Q X Q^T (PAPER.md:363 Vec
    convention); with arr[b] = X_b^T this is B arr C^T + alpha Q arr Q^T.
    """
    if H.dim == 1:
        return X @ H.A[l].T
    B, C, Q = H.Bf[l], H.Cf[l], H.Q[l]
    return np.matmul(np.matmul(B, X), C.T) + H.alpha * np.matmul(np.matmul(Q, X), Q.T)


def restrict(H: Hierarchy, l: int, X: np.ndarray) -> np.ndarray:
    """I_l^{l+1} (2D: hat I = I (x) I, i.e. R X R^T on the matrix)."""
    R = H.R[l]
    if H.dim == 1:
        return X @ R.T
    return np.matmul(np.matmul(R, X), R.T)


def interpolate(H: Hierarchy, l: int, X: np.ndarray) -> np.ndarray:
    """I_{l+1}^l (2D: P X P^T)."""
    P = H.P[l]
    if H.dim == 1:
        return X @ P.T
    return np.matmul(np.matmul(P, X), P.T)


# ==========================================================================
# Coarsest solve: LU with partial pivoting (Gaussian elimination)
# ==========================================================================

def lu_factor(A: np.ndarray):
    """Doolittle LU with partial pivoting: P A = L U, stored compactly."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    piv = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        if A[p, k] == 0.0:
            raise np.linalg.LinAlgError(f"singular coarse operator at pivot {k}")
        if p != k:
            A[[k, p]] = A[[p, k]]
            piv[[k, p]] = piv[[p, k]]
        A[k + 1:, k] /= A[k, k]
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    return A, piv


def lu_solve(lu, Y: np.ndarray) -> np.ndarray:
    """Solve A X^T = Y^T for a batch of right-hand sides (rows of Y)."""
    LU, piv = lu
    n = LU.shape[0]
    Z = np.array(Y, dtype=np.float64)[:, piv].T.copy()      # n x B
    for i in range(n):                                       # forward, unit lower
        Z[i] -= LU[i, :i] @ Z[:i]
    for i in range(n - 1, -1, -1):                           # backward, upper
        Z[i] = (Z[i] - LU[i, i + 1:] @ Z[i + 1:]) / LU[i, i]
    return Z.T


def coarse_solve(H: Hierarchy, Y: np.ndarray) -> np.ndarray:
    """x_L = (A^{(L)})^{-1} y_L (Alg 3; Alg 4 P:382 with Mat/Vec)."""
    if H.dim == 1:
        return lu_solve(H.lu, Y)
    B, n = Y.shape[0], Y.shape[-1]
    return lu_solve(H.lu, Y.reshape(B, n * n)).reshape(B, n, n)


# ==========================================================================
# Masks and level filters (readings R5, R6)
# ==========================================================================

def mask_fn_1d(phi, l: int):
    """m_l(phi) = sqrt(|phi| / (pi/2^{l-1})) on [-pi/2^{l-1}, pi/2^{l-1}], else 0
    (|phi| per R5, as the 2D definition P:406 writes it)."""
    phi = np.asarray(phi, dtype=np.float64)
    a = math.pi / 2 ** (l - 1)
    return np.where(np.abs(phi) <= a, np.sqrt(np.abs(phi) / a), 0.0)


def mask_fn_2d(phi1, phi2, l: int):
    """hat m_l(phi1, phi2)."""
    a = math.pi / 2 ** (l - 1)
    m = np.maximum(np.abs(phi1), np.abs(phi2))
    inside = (np.abs(phi1) <= a) & (np.abs(phi2) <= a)
    return np.where(inside, np.sqrt(m / a), 0.0)


def level_mask(n_l: int, dim: int) -> np.ndarray:
    """m'_l: m_l sampled uniformly over the level's visible band with n_l points
    (P:306), on the points phi_k = (2k - n_l) a / n_l (the paper's own sampling,
    P:87, scaled to a = pi/2^{l-1}).  Returned in natural DFT order (R5): bin j
    holds the sample at centred index k = (j + n_l/2) mod n_l.  The level-local
    profile is the same at every level, so l = 1 is used with a = pi.
    """
    k = np.arange(n_l)
    phi_centred = (2 * k - n_l) * math.pi / n_l
    if dim == 1:
        m_centred = mask_fn_1d(phi_centred, 1)
        return np.roll(m_centred, -(n_l // 2))           # centred -> natural order
    m_c = mask_fn_2d(phi_centred[:, None], phi_centred[None, :], 1)
    return np.roll(np.roll(m_c, -(n_l // 2), axis=0), -(n_l // 2), axis=1)


def level_filter(H: Hierarchy, l: int, Hv: np.ndarray) -> np.ndarray:
    """F'_l(h) = Re(DFT^{-1}(m'_l (.) DFT(h))) (2D P:415)."""
    m = H.masks[l]
    if H.dim == 1:
        return np.real(np.fft.ifft(m[None, :] * np.fft.fft(Hv, axis=-1), axis=-1))
    return np.real(np.fft.ifft2(m[None, :, :] * np.fft.fft2(Hv, axes=(-2, -1)), axes=(-2, -1)))


# ==========================================================================
# CNN smoother N_theta (reading R7)
# ==========================================================================

def conv_same(x: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Cross-correlation with zero 'same' padding, stride 1, plus bias.

    1D: x [B][Cin][n], W [Cout][Cin][k]:
        y[b,o,i] = bias[o] + sum_c sum_t W[o,c,t] x[b,c,i+t-k//2]
    2D: x [B][Cin][n2][n1], W [Cout][Cin][k2][k1]:
        y[b,o,i2,i1] = bias[o] + sum_c sum_{t2,t1} W[o,c,t2,t1] x[b,c,i2+t2-k//2,i1+t1-k//2]
    One channel contraction (tensordot) per tap.
    """
    k = W.shape[-1]
    p = k // 2
    if x.ndim == 3:
        Bn, Ci, n = x.shape
        xp = np.zeros((Bn, Ci, n + 2 * p))
        xp[:, :, p:p + n] = x
        y = np.zeros((Bn, W.shape[0], n)) + b[None, :, None]
        for t in range(k):
            # contraction over input channels c of W[o, c, t] and x[b, c, i + t - k//2]
            y += np.tensordot(W[:, :, t], xp[:, :, t:t + n], axes=([1], [1])).transpose(1, 0, 2)
        return y
    Bn, Ci, n2, n1 = x.shape
    xp = np.zeros((Bn, Ci, n2 + 2 * p, n1 + 2 * p))
    xp[:, :, p:p + n2, p:p + n1] = x
    y = np.zeros((Bn, W.shape[0], n2, n1)) + b[None, :, None, None]
    for t2 in range(k):
        for t1 in range(k):
            # contraction over c of W[o, c, t2, t1] and x[b, c, i2 + t2 - k//2, i1 + t1 - k//2]
            y += np.tensordot(W[:, :, t2, t1], xp[:, :, t2:t2 + n2, t1:t1 + n1],
                              axes=([1], [1])).transpose(1, 0, 2, 3)
    return y


def cnn_forward(layers, u: np.ndarray) -> np.ndarray:
    """N_theta(u): conv, ReLU between layers, no activation after the last (R7).
    u: 1D [B][n] or 2D [B][n2][n1]; returns the same shape."""
    z = u[:, None]
    for i, (W, b) in enumerate(layers):
        z = conv_same(z, W, b)
        if i + 1 < len(layers):
            z = np.maximum(z, 0.0)
    return z[:, 0]


# ==========================================================================
# FNO smoother (section 3.1; Appendix A; Table 6)
# ==========================================================================
# N(u) = proj o f_L o ... o f_1 o lift (u), with the Fourier layer (Appendix A)
#   f(Z) = sigma( DFT^{-1}( R (.) DFT(Z) ) + W Z + B ),
# R a learnable complex c x c channel mixing applied to the k lowest frequencies only (the others
# are zeroed), W a convolution (kernel size per Table 6), B a bias, sigma = GELU (reading R24:
# the paper leaves sigma unnamed; GELU is the activation of the FNO it builds on), lift / proj
# pointwise fully connected layers 1 -> c and c -> 1.

def fno_params(dim: int, c: int, L: int, k: int, ks: int, flat: np.ndarray) -> dict:
    """Unpack the flat fp32 parameter vector (nmg_inputs.fno_param_shapes order) to fp64."""
    p = {"dim": dim, "c": c, "L": L, "k": k, "ks": ks}
    o = 0
    flat = np.asarray(flat, np.float64)

    def take(sh):
        nonlocal o
        m = int(np.prod(sh))
        v = flat[o:o + m].reshape(sh)
        o += m
        return v
    p["lift_w"], p["lift_b"] = take((c, 1))[:, 0], take((c,))
    spec = (k, c, c, 2) if dim == 1 else (2 * k, k, c, c, 2)
    conv = (c, c, ks) if dim == 1 else (c, c, ks, ks)
    p["layers"] = []
    for _ in range(L):
        Rr = take(spec)
        p["layers"].append((Rr[..., 0] + 1j * Rr[..., 1], take(conv), take((c,))))
    p["proj_w"], p["proj_b"] = take((1, c))[0], take((1,))[0]
    assert o == flat.size
    return p


def gelu(z: np.ndarray) -> np.ndarray:
    """sigma(z) = z Phi(z) = z (1 + erf(z / sqrt 2)) / 2 (exact GELU)."""
    from scipy.special import erf
    return 0.5 * z * (1.0 + erf(z / math.sqrt(2.0)))


def spectral_conv(z: np.ndarray, R: np.ndarray, k: int) -> np.ndarray:
    """DFT^{-1}(R (.) DFT(z)) with R acting on the k lowest modes per axis only.

    1D: z [B][c][n]; Z = rfft(z)[..., :k]; Y[b,o,m] = sum_c Z[b,c,m] R[m,c,o]; irfft with the
        modes >= k zero (real output, length n).
    2D: z [B][c][n2][n1]; Z = rfft2(z) (half spectrum along i1); the kept modes are i1-modes
        0..k-1 and i2-modes 0..k-1 and n-k..n-1 (R[j2, m1] with j2 < k the low and j2 >= k the
        high i2-modes); irfft2 with every other mode zero.
    """
    if z.ndim == 3:
        n = z.shape[-1]
        Z = np.fft.rfft(z, axis=-1)[..., :k]
        Y = np.einsum("bcm,mco->bom", Z, R)
        Yp = np.zeros((z.shape[0], R.shape[-1], n // 2 + 1), dtype=complex)
        Yp[..., :k] = Y
        return np.fft.irfft(Yp, n=n, axis=-1)
    n2, n1 = z.shape[-2:]
    Z = np.fft.rfft2(z, axes=(-2, -1))
    Zk = np.concatenate([Z[:, :, :k, :k], Z[:, :, n2 - k:, :k]], axis=2)     # [B][c][2k][k]
    Y = np.einsum("bcjm,jmco->bojm", Zk, R)
    Yp = np.zeros((z.shape[0], R.shape[-1], n2, n1 // 2 + 1), dtype=complex)
    Yp[:, :, :k, :k] = Y[:, :, :k]
    Yp[:, :, n2 - k:, :k] = Y[:, :, k:]
    return np.fft.irfft2(Yp, s=(n2, n1), axes=(-2, -1))


def fno_forward(p: dict, u: np.ndarray) -> np.ndarray:
    """N_theta(u) of the FNO smoother; u 1D [B][n] or 2D [B][n2][n1] -> same shape."""
    ex = (None, slice(None)) + (None,) * (u.ndim - 1)
    z = p["lift_w"][ex] * u[:, None] + p["lift_b"][ex]
    for R, W, bias in p["layers"]:
        z = gelu(spectral_conv(z, R, p["k"]) + conv_same(z, W, bias))
    return np.tensordot(p["proj_w"], z, axes=([0], [1])) + p["proj_b"]


def smoother_forward(theta, u: np.ndarray) -> np.ndarray:
    """N_theta(u) for either smoother family (CNN: list of layers; FNO: dict)."""
    return fno_forward(theta, u) if isinstance(theta, dict) else cnn_forward(theta, u)


# ==========================================================================
# NMGF cycle (Alg 3 P:315-339 / Alg 4)
# ==========================================================================

def rhs_norm(X: np.ndarray) -> np.ndarray:
    """||b_l||_2 per RHS; Frobenius for 2D matrices (R10)."""
    return np.sqrt((X.reshape(X.shape[0], -1) ** 2).sum(axis=1))


def smoothing_step(H: Hierarchy, l: int, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """One neural smoothing step at level l (0-based), Alg 3 P:327-329:
        b = y - A x;  h = N(b/||b||) ||b||;  x <- x + F'_l(h)   (F' off: x + h, Alg 2)
    ||b|| = 0 gives h = 0 (R10 guard)."""
    b = y - apply_A(H, l, x)
    s = rhs_norm(b)
    shape = (-1,) + (1,) * (b.ndim - 1)
    safe = np.where(s > 0, s, 1.0).reshape(shape)
    hv = smoother_forward(H.weights[l], b / safe) * safe
    hv = np.where(s.reshape(shape) > 0, hv, 0.0)
    if H.level_filter:
        hv = level_filter(H, l, hv)
    return x + hv


def nmgf_cycle(H: Hierarchy, x0: np.ndarray, y: np.ndarray, l: int = 0) -> np.ndarray:
    """NMGF(x*, y, A^{(l)}, l, L) with nu1 pre- and nu2 post-smoothing steps (R9).

    l = L: exact solve.  Otherwise:
      x = S_l^{nu1}(x*, y);  y_{l+1} = I_l^{l+1}(y - A x);
      x = x + I_{l+1}^l NMGF(0, y_{l+1}, l+1);  x = S_l^{nu2}(x, y).
    """
    if l == H.levels - 1:
        return coarse_solve(H, y)
    x = x0
    for _ in range(H.nu1):
        x = smoothing_step(H, l, x, y)
    r = y - apply_A(H, l, x)
    yc = restrict(H, l, r)
    e = nmgf_cycle(H, np.zeros_like(yc), yc, l + 1)
    x = x + interpolate(H, l, e)
    for _ in range(H.nu2):
        x = smoothing_step(H, l, x, y)
    return x


@dataclass
class SolveReport:
    """SPEC SolveReport analogue: per-RHS cycle counts and residual history."""
    cycles: np.ndarray
    converged: np.ndarray
    history: np.ndarray          # [nrhs][max_cycles+1], NaN after freezing
    x: np.ndarray


def relative_residual(H: Hierarchy, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    ny = rhs_norm(y)
    nr = rhs_norm(y - apply_A(H, 0, x))
    return np.where(ny > 0, nr / np.where(ny > 0, ny, 1.0), 0.0)


def solve(H: Hierarchy, y: np.ndarray, tol: float = 1e-6, max_cycles: int = 50,
          x0: Optional[np.ndarray] = None, freeze: bool = True) -> SolveReport:
    """Outer iteration x^tau = NMGF(x^{tau-1}, y), x^0 = 0; per RHS stop
    at the first relative residual <= tol; converged RHS are frozen."""
    B = y.shape[0]
    x = np.zeros_like(y) if x0 is None else np.array(x0, dtype=np.float64)
    hist = np.full((B, max_cycles + 1), np.nan)
    rho = relative_residual(H, x, y)
    hist[:, 0] = rho
    active = ~(rho <= tol) if freeze else np.ones(B, bool)
    cycles = np.zeros(B, np.int32)
    for tau in range(1, max_cycles + 1):
        if not active.any():
            break
        idx = np.nonzero(active)[0]
        xn = nmgf_cycle(H, x[idx], y[idx])
        if not np.all(np.isfinite(xn)):
            bad = idx[np.nonzero(~np.isfinite(xn.reshape(len(idx), -1)).all(axis=1))[0][0]]
            raise FloatingPointError(f"non-finite iterate at cycle {tau}, rhs {bad}")
        x[idx] = xn
        rho_a = relative_residual(H, xn, y[idx])
        hist[idx, tau] = rho_a
        cycles[idx] = tau
        if freeze:
            active[idx[rho_a <= tol]] = False
    converged = np.nan_to_num(hist, nan=np.inf).min(axis=1) <= tol
    return SolveReport(cycles=cycles, converged=converged, history=hist, x=x)


# ==========================================================================
# Oracle-only extras (never on the GPU hot path)
# ==========================================================================

def weighted_jacobi(A: np.ndarray, x: np.ndarray, y: np.ndarray, omega: float) -> np.ndarray:
    """x <- x + omega D^{-1}(y - A x), D = diag(A) (section 2.2)."""
    d = np.diag(A)
    return x + omega * (y - x @ A.T) / d[None, :]


def dense_operator_2d(H: Hierarchy, l: int) -> np.ndarray:
    """Explicit hat A^{(l)} on column-major Vec (small n only; pin P2)."""
    return np.kron(H.Bf[l], H.Cf[l]) + H.alpha * np.kron(H.Q[l], H.Q[l])
