"""Builds the same problem on both sides (oracle and CUDA path) from the shared
seeded inputs.  The two sides share nothing else."""
import numpy as np

import nmg_inputs as ni


def weights_for(cfg, kind, alpha=None):
    if kind == "seed":
        return ni.weights_seed(cfg)
    if kind == "lin":
        return ni.weights_lin(cfg, alpha=alpha)
    if kind == "zero":
        return ni.weights_zero(cfg)
    raise ValueError(kind)


def oracle_hierarchy(cfg, factors, weights, level_filter=True):
    from oracle import nmg_oracle as O
    H = O.build_hierarchy(cfg.dim, factors, cfg.alpha, cfg.levels, nu1=cfg.nu1, nu2=cfg.nu2,
                          level_filter=level_filter)
    for l, w in enumerate(weights):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    return H


def gpu_hierarchy(cfg, factors, weights, max_rhs, level_filter=True, **kw):
    import paper_2603_01064_b200 as nmg
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, factors, nu1=cfg.nu1, nu2=cfg.nu2,
                      level_filter=level_filter, max_rhs=max_rhs, **kw)
    for l, w in enumerate(weights):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    return h


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0)


def history_close(h_gpu, h_or, tol=1e-3, floor=1e-6):
    """Per-cycle residual histories within `tol` relative while the oracle residual >= floor."""
    h_gpu = np.asarray(h_gpu)
    h_or = np.asarray(h_or)
    m = np.isfinite(h_or) & (h_or >= floor)
    if not m.any():
        return True, 0.0
    err = np.abs(h_gpu[m] - h_or[m]) / h_or[m]
    return bool(err.max() <= tol), float(err.max())
