"""Pins for the fp64 oracle (run with -m "not gpu").

Each test pins a piece of oracle/nmg_oracle.py to something other than
itself: a value the paper prints (tests/golden/), a closed form, a library
routine of a different provenance (torch conv, numpy dense solve), an
invariant of the algorithm, or brute force on tiny inputs.  Pin ids P1..P15
follow DESIGN.md "Pins".
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import nmg_inputs as ni
from oracle import nmg_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _hier(cfg, weights="seed", **kw):
    f = ni.operator_factors(cfg)
    H = O.build_hierarchy(cfg.dim, f, cfg.alpha, cfg.levels, nu1=cfg.nu1, nu2=cfg.nu2, **kw)
    if weights == "seed":
        W = ni.weights_seed(cfg)
    elif weights == "lin":
        W = ni.weights_lin(cfg)
    elif weights == "zero":
        W = ni.weights_zero(cfg)
    else:
        W = weights
    for l, w in enumerate(W):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    return H, f


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line.split())
    return rows


# ----------------------------------------------------------------- P1, P13
def test_P1_operator_spd_and_symmetric():
    """A = K^T K + alpha I is bitwise symmetric and SPD with lambda_min >= alpha."""
    for cfg in (ni.CONFIGS[0], ni.CONFIGS[1].replace(n=512)):
        (G,) = ni.operator_factors(cfg)
        A = G + cfg.alpha * np.eye(cfg.n)
        assert np.array_equal(A, A.T)
        lam = np.linalg.eigvalsh(A)
        assert lam[0] >= cfg.alpha * (1 - 1e-10)
        np.linalg.cholesky(A)
    H, _ = _hier(ni.CONFIGS[0])
    for A in H.A:            # Galerkin keeps SPD (R = P^T/2)
        assert np.allclose(A, A.T, rtol=0, atol=1e-15 * np.abs(A).max())
        assert np.linalg.eigvalsh(A)[0] > 0


def test_P13_kernel_quadrature_normalisation():
    """K rows integrate the unit-mass Gaussian: interior row sums -> 1, ends ~ 1/2."""
    K = ni.gaussian_kernel_1d(256, 0.05)
    assert abs(K[128].sum() - 1.0) < 1e-9
    assert 0.5 < K[0].sum() < 0.53 and 0.5 < K[-1].sum() < 0.53


# ----------------------------------------------------------------- P3 transfers
@pytest.mark.parametrize("n_c", [2, 4, 8, 64])
def test_P3_transfers(n_c):
    P = O.interpolation_matrix(n_c)
    R = O.restriction_matrix(2 * n_c)
    assert np.array_equal(R, 0.5 * P.T)                # variational pair, bitwise (dyadic)
    assert np.array_equal(P @ np.ones(n_c), np.ones(2 * n_c))
    assert np.array_equal(R @ np.ones(2 * n_c), np.ones(n_c))
    # exact on linear functions away from the clamped ends: coarse centres
    # T_j=(j+1/2)/n_c, fine centres t_i=(i+1/2)/(2 n_c)
    T = (np.arange(n_c) + 0.5) / n_c
    t = (np.arange(2 * n_c) + 0.5) / (2 * n_c)
    lin = P @ (3.0 * T - 1.0)
    assert np.allclose(lin[1:-1], 3.0 * t[1:-1] - 1.0, rtol=0, atol=1e-15)


def test_P3_restriction_rows_closed_form():
    R8 = O.restriction_matrix(8) * 8
    assert R8[0].tolist() == [4, 3, 1, 0, 0, 0, 0, 0]
    assert R8[1].tolist() == [0, 1, 3, 3, 1, 0, 0, 0]
    assert R8[3].tolist() == [0, 0, 0, 0, 0, 1, 3, 4]


# ----------------------------------------------------------------- P4, P5 masks / filter
def test_P4_level_mask_golden():
    rows = _read_golden("level_mask_P289_P306.txt")
    m1 = O.level_mask(8, 1)
    want = np.array([float(Fraction(v)) for v in rows[0]])
    assert np.allclose(m1 ** 2, want, rtol=0, atol=1e-15)
    m2 = O.level_mask(4, 2)
    want2 = np.array([[float(Fraction(v)) for v in r] for r in rows[1:5]])
    assert np.allclose(m2 ** 2, want2, rtol=0, atol=1e-15)


def test_P5_mask_semantics_paper():
    """maximum 1 at |phi| = pi/2^{l-1}, -> 0 as phi -> 0, 0 outside the band."""
    for l in (1, 2, 3):
        a = math.pi / 2 ** (l - 1)
        assert O.mask_fn_1d(a, l) == 1.0 and O.mask_fn_1d(-a, l) == 1.0
        assert O.mask_fn_1d(0.0, l) == 0.0
    assert O.mask_fn_1d(math.pi, 2) == 0.0
    assert abs(O.mask_fn_1d(math.pi / 4, 2) - math.sqrt(0.5)) < 1e-15
    assert O.mask_fn_2d(math.pi, 0.0, 1) == 1.0
    assert O.mask_fn_2d(math.pi, math.pi / 2, 2) == 0.0


def _closed_form_filter_matrix(n):
    """F' as a dense circulant: c_j = (1/n) sum_k m[k] cos(2 pi j k / n),
    m[k] = sqrt(2 min(k, n-k)/n) (R5 closed form)."""
    k = np.arange(n)
    m = np.sqrt(2.0 * np.minimum(k, n - k) / n)
    j = np.arange(n)
    c = (m[None, :] * np.cos(2 * math.pi * np.outer(j, k) / n)).sum(1) / n
    return np.array([[c[(i - jj) % n] for jj in range(n)] for i in range(n)]), m


def test_P4_filter_closed_form_1d():
    n = 32
    cfg = ni.CONFIGS[0].replace(n=n, levels=2)
    H, _ = _hier(cfg)
    Cm, m = _closed_form_filter_matrix(n)
    X = np.random.default_rng(5).standard_normal((3, n))
    assert np.allclose(O.level_filter(H, 0, X), X @ Cm.T, rtol=0, atol=1e-14)
    assert np.allclose(Cm, Cm.T, atol=1e-15)
    for kk in (0, 1, 5, 16):
        mode = np.cos(2 * math.pi * kk * np.arange(n) / n)[None]
        assert np.allclose(O.level_filter(H, 0, mode), m[kk] * mode, atol=1e-14)
    spec = np.fft.ifft(O.level_mask(n, 1) * np.fft.fft(X, axis=-1), axis=-1)
    assert np.abs(spec.imag).max() < 1e-14


def test_P4_filter_closed_form_2d():
    n = 8
    cfg = ni.CONFIGS[2].replace(n=n, levels=2)
    H, _ = _hier(cfg)
    k = np.arange(n)
    a = 2.0 * np.minimum(k, n - k) / n
    M = np.sqrt(np.maximum(a[:, None], a[None, :]))
    X = np.random.default_rng(6).standard_normal((2, n, n))
    # brute-force DFT2 sums
    w = np.exp(-2j * math.pi * np.outer(k, k) / n)
    Xh = np.einsum('pi,bij,qj->bpq', w, X, w)
    back = np.einsum('pi,bij,qj->bpq', np.conj(w), M[None] * Xh, np.conj(w)).real / (n * n)
    assert np.allclose(O.level_filter(H, 0, X), back, rtol=0, atol=1e-13)


# ----------------------------------------------------------------- CNN vs torch (library conv)
def test_cnn_matches_torch_conv_1d():
    torch = pytest.importorskip("torch")
    cfg = ni.CONFIGS[0]
    layers = ni.unflatten_params(cfg, ni.weights_seed(cfg)[0])
    u = np.random.default_rng(3).standard_normal((4, 40))
    z = torch.tensor(u[:, None])
    for i, (W, b) in enumerate(layers):
        z = torch.nn.functional.conv1d(z, torch.tensor(W.astype(np.float64)),
                                       torch.tensor(b.astype(np.float64)), padding=cfg.ksize // 2)
        if i + 1 < len(layers):
            z = torch.relu(z)
    ours = O.cnn_forward([(w.astype(np.float64), b.astype(np.float64)) for w, b in layers], u)
    assert np.allclose(ours, z[:, 0].numpy(), rtol=1e-13, atol=1e-13)


def test_cnn_matches_torch_conv_2d():
    torch = pytest.importorskip("torch")
    cfg = ni.CONFIGS[2].replace(channels=6)
    layers = ni.unflatten_params(cfg, ni.weights_seed(cfg)[0])
    u = np.random.default_rng(4).standard_normal((2, 9, 11))
    z = torch.tensor(u[:, None])
    for i, (W, b) in enumerate(layers):
        z = torch.nn.functional.conv2d(z, torch.tensor(W.astype(np.float64)),
                                       torch.tensor(b.astype(np.float64)), padding=1)
        if i + 1 < len(layers):
            z = torch.relu(z)
    ours = O.cnn_forward([(w.astype(np.float64), b.astype(np.float64)) for w, b in layers], u)
    assert np.allclose(ours, z[:, 0].numpy(), rtol=1e-13, atol=1e-13)


def test_cnn_relu_hand_case():
    """Hand-computed: identity-ish 3-tap filters with negative values and a bias
    that the ReLU clips; zero padding at both ends."""
    W0 = np.zeros((1, 1, 3)); W0[0, 0] = [1.0, 0.0, 0.0]       # y[i] = x[i-1]
    b0 = np.array([0.5])
    W1 = np.zeros((1, 1, 3)); W1[0, 0] = [0.0, 0.0, 2.0]       # y[i] = 2 z[i+1]
    b1 = np.array([-1.0])
    u = np.array([[1.0, -2.0, 3.0, -4.0]])
    # layer0: [0, 1, -2, 3] + 0.5 -> relu -> [0.5, 1.5, 0, 3.5]
    # layer1: 2*[1.5, 0, 3.5, 0] - 1 = [2, -1, 6, -1]
    out = O.cnn_forward([(W0, b0), (W1, b1)], u)
    assert out.tolist() == [[2.0, -1.0, 6.0, -1.0]]


def test_smoothing_step_normalisation():
    """h = N(b/||b||_2) ||b||_2 with a non-homogeneous N (bias), and F' off/on."""
    cfg = ni.CONFIGS[0].replace(n=16, levels=2)
    H, _ = _hier(cfg, level_filter=False)
    W = np.zeros((1, 1, 1)); W[0, 0, 0] = 1.0
    H.weights[0] = [(W, np.array([0.25]))]      # N(u) = u + 1/4
    x = np.zeros((2, 16))
    y = np.random.default_rng(7).standard_normal((2, 16))
    out = O.smoothing_step(H, 0, x, y)
    s = np.linalg.norm(y, axis=1, keepdims=True)
    assert np.allclose(out, (y / s + 0.25) * s, rtol=1e-15, atol=1e-15)
    out0 = O.smoothing_step(H, 0, x, np.zeros_like(y))            # ||b|| = 0 guard
    assert np.array_equal(out0, np.zeros_like(y))


# ----------------------------------------------------------------- coarse solve
def test_lu_solve_against_numpy():
    rng = np.random.default_rng(8)
    A = rng.standard_normal((40, 40)) + 40 * np.eye(40)
    Y = rng.standard_normal((5, 40))
    X = O.lu_solve(O.lu_factor(A), Y)
    assert np.allclose(X, np.linalg.solve(A, Y.T).T, rtol=1e-12, atol=1e-12)
    A2 = np.array([[0.0, 1.0], [2.0, 0.0]])            # needs pivoting
    assert np.allclose(O.lu_solve(O.lu_factor(A2), np.array([[3.0, 4.0]])), [[2.0, 3.0]])


def test_P6_single_level_is_exact_solve():
    cfg = ni.CONFIGS[0].replace(n=64, levels=1)
    H, f = _hier(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=3)
    x = O.nmgf_cycle(H, np.zeros_like(y), y)
    assert O.relative_residual(H, x, y).max() <= 1e-12


# ----------------------------------------------------------------- P7 W_zero
@pytest.mark.parametrize("dim", [1, 2])
def test_P7_zero_smoother_is_coarse_projection(dim):
    cfg = (ni.CONFIGS[0].replace(n=64, levels=3) if dim == 1
           else ni.CONFIGS[2].replace(n=16, levels=3, channels=4))
    H, f = _hier(cfg, weights="zero")
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=2)
    x = O.nmgf_cycle(H, np.zeros_like(y), y)
    r = y - O.apply_A(H, 0, x)
    rc = O.restrict(H, 1, O.restrict(H, 0, r))
    yc = O.restrict(H, 1, O.restrict(H, 0, y))
    assert np.abs(rc).max() <= 1e-12 * np.abs(yc).max()
    x2 = O.nmgf_cycle(H, x, y)
    assert np.abs(x2 - x).max() <= 1e-10 * np.abs(x).max()


# ----------------------------------------------------------------- P8 two-grid identity
def _toeplitz_corr(g, n):
    """Zero-padded cross-correlation matrix: (T u)[i] = sum_t g[t] u[i+t-k//2]."""
    k = len(g)
    T = np.zeros((n, n))
    for i in range(n):
        for t in range(k):
            j = i + t - k // 2
            if 0 <= j < n:
                T[i, j] += g[t]
    return T


def _cycle_matrix_1d(H, n):
    return np.stack([O.nmgf_cycle(H, e[None], np.zeros((1, n)))[0] for e in np.eye(n)], axis=1)


@pytest.mark.parametrize("levels", [2, 3])
def test_P8_two_grid_error_propagation_1d(levels):
    n = 32
    cfg = ni.CONFIGS[0].replace(n=n, levels=levels)
    H, f = _hier(cfg, weights="lin")
    A = f[0] + cfg.alpha * np.eye(n)
    # independent construction: level operators, linear smoother C_l G_l, recursion
    Als = [A]
    for q in range(levels - 1):
        Als.append(O.restriction_matrix(n >> q) @ Als[-1] @ O.interpolation_matrix(n >> (q + 1)))

    def E(l):   # error propagator of NMGF at level l (0-based), nu1 = nu2 = 1
        nl = n >> l
        G = (1.0 / cfg.alpha) * _toeplitz_corr(ni.default_g1(cfg), nl)  # delta layers = identity
        Cm, _ = _closed_form_filter_matrix(nl)
        S = np.eye(nl) - Cm @ G @ Als[l]
        inner = np.linalg.inv(Als[l + 1])
        if l + 1 < levels - 1:                  # coarse "solve" is itself a cycle from 0
            inner = (np.eye(nl // 2) - E(l + 1)) @ inner
        Pm, Rm = O.interpolation_matrix(nl // 2), O.restriction_matrix(nl)
        return S @ (np.eye(nl) - Pm @ inner @ Rm @ Als[l]) @ S

    got = _cycle_matrix_1d(H, n)
    want = E(0)
    assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()


def test_P8_two_grid_error_propagation_2d():
    n = 8
    cfg = ni.CONFIGS[2].replace(n=n, levels=2, channels=2, kernel="gauss_cos", sigma=0.15)
    H, f = _hier(cfg, weights="lin")
    N = n * n
    Bf, Cf = f
    A = np.kron(Bf, Cf) + cfg.alpha * np.eye(N)
    # 2D zero-padded correlation of the 3x3 g1 on column-major Vec (index i1 + n i2)
    g1 = ni.default_g1(cfg)
    G = np.zeros((N, N))
    for i2 in range(n):
        for i1 in range(n):
            for t2 in range(3):
                for t1 in range(3):
                    j2, j1 = i2 + t2 - 1, i1 + t1 - 1
                    if 0 <= j2 < n and 0 <= j1 < n:
                        G[i1 + n * i2, j1 + n * j2] += g1[t2, t1]
    G /= cfg.alpha
    k = np.arange(n)
    a = 2.0 * np.minimum(k, n - k) / n
    M = np.sqrt(np.maximum(a[:, None], a[None, :]))     # [k2][k1]
    Cm = np.zeros((N, N))
    for i2 in range(n):
        for i1 in range(n):
            for j2 in range(n):
                for j1 in range(n):
                    ph = np.cos(2 * math.pi * (np.outer(k, np.ones(n)) * (i2 - j2) +
                                               np.outer(np.ones(n), k) * (i1 - j1)) / n)
                    Cm[i1 + n * i2, j1 + n * j2] = (M * ph).sum() / N
    S = np.eye(N) - Cm @ G @ A
    R1, P1 = O.restriction_matrix(n), O.interpolation_matrix(n // 2)
    R, P = np.kron(R1, R1), np.kron(P1, P1)
    Ac = R @ A @ P
    E = S @ (np.eye(N) - P @ np.linalg.inv(Ac) @ R @ A) @ S
    got = np.stack([O.nmgf_cycle(H, e.reshape(1, n, n), np.zeros((1, n, n)))[0].reshape(N)
                    for e in np.eye(N)], axis=1)
    assert np.abs(got - E).max() <= 1e-10 * np.abs(E).max()


# ----------------------------------------------------------------- P2 Kronecker / Galerkin
@pytest.mark.parametrize("kernel", ["gauss", "gauss_cos"])
def test_P2_kronecker_apply_and_galerkin_2d(kernel):
    # gauss_cos has B != C, so a swapped or transposed factor is caught
    cfg = ni.CONFIGS[2].replace(n=16, levels=3, channels=2, kernel=kernel, sigma=0.1)
    H, f = _hier(cfg)
    rng = np.random.default_rng(9)
    Ahat = np.kron(f[0], f[1]) + cfg.alpha * np.eye(256)
    for l in range(3):
        nl = H.n[l]
        X = rng.standard_normal((2, nl, nl))
        dense = O.dense_operator_2d(H, l)
        want = (X.reshape(2, -1) @ dense.T).reshape(2, nl, nl)
        assert np.allclose(O.apply_A(H, l, X), want, rtol=0, atol=1e-14 * np.abs(want).max())
    # Galerkin in dense form equals the Kronecker-factor chain
    R1, P1 = O.restriction_matrix(16), O.interpolation_matrix(8)
    Ac = np.kron(R1, R1) @ Ahat @ np.kron(P1, P1)
    assert np.allclose(Ac, O.dense_operator_2d(H, 1), rtol=0, atol=1e-15 * np.abs(Ac).max())
    assert np.allclose(O.dense_operator_2d(H, 0), Ahat, rtol=0, atol=0)


def test_cfg4_separable_matches_direct_truncated_convolution():
    """Reading R17: the cos-modulated Gaussian is K_(2) (x) K_(1); check the
    Kronecker G-apply against a direct truncated 2D convolution on sampled rows."""
    cfg = ni.CONFIGS[4].replace(n=128)
    K_a = ni.gaussian_kernel_1d(cfg.n, cfg.sigma, cos_mod=0.3)
    K_b = ni.gaussian_kernel_1d(cfg.n, cfg.sigma)
    off, w = ni.truncated_kernel_2d_cfg4(cfg.n, cfg.sigma)
    X = np.random.default_rng(10).standard_normal((cfg.n, cfg.n))    # [i2][i1]
    KX = K_b @ X @ K_a.T                                               # Vec(K_a X K_b^T)
    for (i2, i1) in [(0, 0), (5, 64), (64, 64), (127, 3)]:
        s = 0.0
        for (o1, o2), wt in zip(off, w):
            j1, j2 = i1 - o1, i2 - o2
            if 0 <= j1 < cfg.n and 0 <= j2 < cfg.n:
                s += wt * X[j2, j1]
        assert abs(s - KX[i2, i1]) <= 1e-11 * np.abs(KX).max()


# ----------------------------------------------------------------- P9 Jacobi
def test_P9_jacobi_smoothing_factor_golden():
    rows = _read_golden("jacobi_reduction_P102.txt")
    n = 64
    for alpha_s, phi_s, red_s in rows:
        alpha, phi = float(alpha_s), float(phi_s) * math.pi
        A = (2 + alpha) * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
        A[0, -1] = A[-1, 0] = -1.0
        e = np.cos(phi * np.arange(n))[None]
        e2 = O.weighted_jacobi(A, e, np.zeros_like(e), 0.5)        # error propagation S e
        mu = (e2 @ e.T / (e @ e.T)).item()
        assert abs((1 - mu) - float(Fraction(red_s))) < 1e-12


def test_P9_jacobi_fails_on_integral_operator():
    """Jacobi damps the smooth (large-eigenvalue) mode of the integral
    operator, not the oscillatory (small-eigenvalue) one."""
    cfg = ni.CONFIGS[0]
    (G,) = ni.operator_factors(cfg)
    A = G + cfg.alpha * np.eye(cfg.n)
    Dinv = 1.0 / np.diag(A)
    rho = np.abs(np.linalg.eigvals(Dinv[:, None] * A)).max()
    lam, V = np.linalg.eigh(A)
    osc, smooth = V[:, 0], V[:, -1]
    assert np.sum(np.diff(np.sign(osc)) != 0) > 50 and np.sum(np.diff(np.sign(smooth)) != 0) <= 1
    f = []
    for v in (osc, smooth):
        e2 = O.weighted_jacobi(A, v[None], np.zeros((1, cfg.n)), 1.0 / rho)
        f.append(abs((e2 @ v).item()))
    assert f[0] > 0.99 and f[1] < 0.1


# ----------------------------------------------------------------- P10, P11, P14, P15
def test_P10_positive_homogeneity_bitwise():
    cfg = ni.CONFIGS[0]
    H, f = _hier(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=3)
    base = O.nmgf_cycle(H, np.zeros_like(y), y)
    for k in (3, -5):
        s = 2.0 ** k
        assert np.array_equal(O.nmgf_cycle(H, np.zeros_like(y), s * y), s * base)


def test_P11_correction_form():
    cfg = ni.CONFIGS[0]
    H, f = _hier(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=3)
    xs = np.random.default_rng(11).standard_normal(y.shape)
    direct = O.nmgf_cycle(H, xs, y)
    corr = xs + O.nmgf_cycle(H, np.zeros_like(y), y - O.apply_A(H, 0, xs))
    assert np.abs(direct - corr).max() <= 1e-11 * np.abs(direct).max()


def test_P14_per_rhs_independence():
    cfg = ni.CONFIGS[0]
    H, f = _hier(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=4)
    batch = O.nmgf_cycle(H, np.zeros_like(y), y)
    for b in range(4):
        one = O.nmgf_cycle(H, np.zeros_like(y[b:b + 1]), y[b:b + 1])[0]
        assert np.abs(one - batch[b]).max() <= 1e-12 * np.abs(batch[b]).max()   # BLAS blocking order


def test_P15_zero_rhs():
    cfg = ni.CONFIGS[0]
    H, f = _hier(cfg)
    rep = O.solve(H, np.zeros((2, cfg.n)), max_cycles=3)
    assert np.array_equal(rep.x, np.zeros((2, cfg.n))) and rep.converged.all()


# ----------------------------------------------------------------- P12 fixed point
def test_P12_fixed_point_is_dense_solve():
    cfg = ni.CONFIGS[0].replace(n=64, levels=3, alpha=1e-2, sigma=0.08)
    H, f = _hier(cfg, weights="lin")
    H.nu2 = 0
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=2)
    rep = O.solve(H, y, tol=1e-13, max_cycles=400)
    assert rep.converged.all()
    A = f[0] + cfg.alpha * np.eye(cfg.n)
    xe = np.linalg.solve(A, y.T).T
    kappa = np.linalg.cond(A)
    assert np.abs(rep.x - xe).max() <= 1e-10 * kappa * np.abs(xe).max()


def test_cfg0_wlin_converges_wseed_stagnates():
    """Sanity of the two weight sets on config 0 (SURVEY App. A.2/A.4 magnitudes)."""
    cfg = ni.CONFIGS[0]
    H, f = _hier(cfg, weights="lin")
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    H.nu2 = 0
    rep = O.solve(H, y, max_cycles=60)
    assert rep.converged.all() and rep.cycles.max() < 60
    H2, _ = _hier(cfg, weights="seed")
    rep2 = O.solve(H2, y, max_cycles=10, freeze=False)
    assert np.all(rep2.history[:, 10] > 1e-4)


# ------------------------------------------------------------------ FNO smoother (NEXT-2)
def _dft_spectral_bruteforce_1d(z, R, k):
    """DFT^{-1}(R (.) DFT(z)) from the DFT definition: Z_m = sum_p z_p e^{-2 pi i m p / n} for the
    kept modes m < k, Y_m = sum_c Z_m[c] R[m, c, o], and the real inverse of the Hermitian
    spectrum that has Y at +m, conj(Y) at -m and zeros elsewhere:
    x_p = (Re Y_0 + 2 sum_{0<m<k} Re(Y_m e^{2 pi i m p / n})) / n."""
    B, c, n = z.shape
    out = np.zeros((B, R.shape[2], n))
    for b in range(B):
        for m in range(k):
            Zm = np.array([sum(z[b, ch, p] * np.exp(-2j * np.pi * m * p / n) for p in range(n)) for ch in range(c)])
            Ym = Zm @ R[m]
            for p in range(n):
                w = 1.0 if m == 0 else 2.0
                out[b, :, p] += w * np.real(Ym * np.exp(2j * np.pi * m * p / n)) / n
    return out


def test_fno_spectral_conv_1d_bruteforce():
    rng = np.random.default_rng(21)
    z = rng.standard_normal((2, 3, 8))
    R = rng.standard_normal((3, 3, 2)) + 1j * rng.standard_normal((3, 3, 2))
    got = O.spectral_conv(z, R, 3)
    want = _dft_spectral_bruteforce_1d(z, R, 3)
    assert np.abs(got - want).max() < 1e-12


def test_fno_spectral_conv_2d_bruteforce():
    """2D: kept modes i1 in {0..k-1} x i2 in {0..k-1} U {n-k..n-1}; brute force over the full
    complex 2D DFT with the Hermitian completion (i1-mode -m1 paired with i2-mode -m2)."""
    rng = np.random.default_rng(22)
    n, k, c = 8, 2, 2
    z = rng.standard_normal((1, c, n, n))
    R = rng.standard_normal((2 * k, k, c, 2)) + 1j * rng.standard_normal((2 * k, k, c, 2))
    got = O.spectral_conv(z, R, k)
    i2 = np.arange(n)[:, None]
    i1 = np.arange(n)[None, :]
    full = np.zeros((2, n, n), dtype=complex)      # full spectrum of the output channels
    for j2 in range(2 * k):
        m2 = j2 if j2 < k else n - 2 * k + j2
        for m1 in range(k):
            E = np.exp(-2j * np.pi * (m2 * i2 + m1 * i1) / n)
            Zm = np.array([(z[0, ch] * E).sum() for ch in range(c)])
            Y = Zm @ R[j2, m1]
            full[:, m2, m1] += Y
            if m1 > 0:      # Hermitian partner of an i1-mode > 0 (not stored in the half spectrum)
                full[:, (-m2) % n, (-m1) % n] += np.conj(Y)
    # the i1-mode-0 column keeps only its real-symmetric part (irfft drops Im of that column's
    # inverse along i1): (Y + conj Y(-m2)) / 2 per i2-mode pair
    col0 = full[:, :, 0].copy()
    full[:, :, 0] = 0.5 * (col0 + np.conj(col0[:, (-np.arange(n)) % n]))
    want = np.zeros((2, n, n))
    for m2 in range(n):
        for m1 in range(n):
            want += np.real(full[:, m2, m1][:, None, None] * np.exp(2j * np.pi * (m2 * i2 + m1 * i1) / n)) / n ** 2
    assert np.abs(got[0] - want).max() < 1e-12


@pytest.mark.parametrize("dim", [1, 2])
def test_fno_forward_vs_torch(dim):
    """The oracle FNO (numpy FFTs, tensordot convs, erf GELU) against an independent torch
    composition (torch.fft, conv1d/conv2d, torch GELU) on seeded weights."""
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    n = 32 if dim == 1 else 16
    c, L, k, ks = (8, 2, 5, 5) if dim == 1 else (6, 2, 3, 3)
    cfg = ni.CONFIGS[0 if dim == 1 else 2].replace(n=n, levels=2)
    flat = ni.fno_weights_seed(cfg, seed=5, width=c)[0]
    c0, L0, k0, ks0 = ni.fno_arch(dim, n, c)
    P = ni.fno_unflatten(dim, c0, L0, k0, ks0, flat)
    p = O.fno_params(dim, c0, L0, k0, ks0, flat)
    rng = np.random.default_rng(3)
    u = rng.standard_normal((2,) + (n,) * dim)
    ours = O.fno_forward(p, u)
    t = lambda a: torch.tensor(np.asarray(a, np.float64))   # noqa: E731
    z = F.linear(t(u)[..., None], t(P["lift_w"]), t(P["lift_b"])).movedim(-1, 1)
    for i in range(L0):
        Rr = t(P[f"spec{i}"])
        Rc = torch.complex(Rr[..., 0], Rr[..., 1])
        if dim == 1:
            Z = torch.fft.rfft(z, dim=-1)[..., :k0]
            Yp = torch.zeros(z.shape[0], c0, n // 2 + 1, dtype=torch.complex128)
            Yp[..., :k0] = torch.einsum("bcm,mco->bom", Z, Rc)
            s = torch.fft.irfft(Yp, n=n, dim=-1)
            w = F.conv1d(z, t(P[f"conv{i}"]), t(P[f"bias{i}"]), padding=ks0 // 2)
        else:
            Z = torch.fft.rfft2(z)
            Yp = torch.zeros(z.shape[0], c0, n, n // 2 + 1, dtype=torch.complex128)
            Yp[:, :, :k0, :k0] = torch.einsum("bcjm,jmco->bojm", Z[:, :, :k0, :k0], Rc[:k0])
            Yp[:, :, n - k0:, :k0] = torch.einsum("bcjm,jmco->bojm", Z[:, :, n - k0:, :k0], Rc[k0:])
            s = torch.fft.irfft2(Yp, s=(n, n))
            w = F.conv2d(z, t(P[f"conv{i}"]), t(P[f"bias{i}"]), padding=ks0 // 2)
        z = F.gelu(s + w)
    ref = (F.linear(z.movedim(1, -1), t(P["proj_w"]), t(P["proj_b"]))[..., 0]).numpy()
    assert np.abs(ours - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
