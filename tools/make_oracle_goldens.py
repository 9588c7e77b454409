#!/usr/bin/env python
"""Writes tests/golden/oracle_*.npz: fp64 ORACLE residual histories / stopping cycles for the
GPU parity tests that run the benchmark's exact launch configurations (full batches).

Calls only oracle/ and the seeded input module nmg_inputs (no CUDA path): the stored values
are the oracle's, so the GPU tests compare against them without re-running the slow oracle
on the GPU box.  Re-run after any change to the oracle's arithmetic or to nmg_inputs.

  1D (BASELINE configs[1], 1024 RHS): sampled RHS incl. the RHS-lane edges of the bench's
     4-lane launch (255/256, 511/512, 767/768):
       * W_seed, alpha in {1e-2, 1e-3, 1e-4}: 10-cycle residual histories;
       * W_lin,  alpha in {1e-2, 1e-3}: solve to relres 1e-6 -> histories + cycles.
  2D (configs[2], [3] at alpha 1e-3 / 1e-4, [4]): the bench's 8-RHS seeded pool (tiled to the
     batch on the GPU), 3-cycle W_seed histories of the first `m` pool members.

  W_train (trainer/nmg_train.py output): oracle solves to 1e-6 with the trained smoothers.

Usage: python tools/make_oracle_goldens.py [which ...]   (which in 1d_seed 1d_lin 2d trained)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nmg_inputs as ni  # noqa: E402
from oracle import nmg_oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
IDX_1D = [0, 1, 127, 128, 255, 256, 257, 500, 511, 512, 513, 767, 768, 769, 1022, 1023]
POOL_2D = {"cfg2": (2, 1e-3, 8), "cfg3_a1e-3": (3, 1e-3, 4), "cfg3_a1e-4": (3, 1e-4, 4), "cfg4": (4, 1e-4, 2)}


def hierarchy(cfg, f, weights):
    H = O.build_hierarchy(cfg.dim, f, cfg.alpha, cfg.levels, nu1=cfg.nu1, nu2=cfg.nu2)
    for l, w in enumerate(weights):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    return H


def one_d_seed():
    out = {"idx": np.array(IDX_1D)}
    for a in ni.ALPHAS[1]:
        cfg = ni.CONFIGS[1].replace(alpha=a)
        f = ni.operator_factors(cfg)
        H = hierarchy(cfg, f, ni.weights_seed(cfg))
        y, _ = ni.make_rhs(cfg, f, a)
        orc = O.solve(H, y[IDX_1D], tol=1e-300, max_cycles=cfg.cycles, freeze=False)
        out[f"hist_{a:g}"] = orc.history
    np.savez_compressed(os.path.join(GOLD, "oracle_cfg1_wseed.npz"), **out)


def one_d_lin():
    out = {"idx": np.array(IDX_1D)}
    for a in (1e-2, 1e-3):
        cfg = ni.CONFIGS[1].replace(alpha=a)
        f = ni.operator_factors(cfg)
        H = hierarchy(cfg, f, ni.weights_lin(cfg))
        y, _ = ni.make_rhs(cfg, f, a)
        orc = O.solve(H, y[IDX_1D], tol=1e-6, max_cycles=100)
        out[f"hist_{a:g}"] = orc.history
        out[f"cycles_{a:g}"] = orc.cycles
        out[f"conv_{a:g}"] = orc.converged
    np.savez_compressed(os.path.join(GOLD, "oracle_cfg1_wlin.npz"), **out)


def trained(cids=(0, 1, 2, 3, 4)):
    """W_train (trainer output, nmg_inputs/trained): oracle solves to 1e-6 -- the
    oracle's confirmation that the trained smoothers converge, and the stopping cycles the GPU
    solve must reproduce.  Config 0: its 8 RHS; 1D: the IDX_1D RHS of the full batch; 2D: 4 pool
    members (cfg 3: 2).  Entries of configs outside `cids` are kept from the existing file."""
    out = {}
    p = os.path.join(GOLD, "oracle_wtrain.npz")
    if os.path.exists(p):
        with np.load(p) as z:
            keep = {k: z[k] for k in z.files if int(k.split("cfg")[1][0]) not in cids}
        out.update(keep)
    for cid in cids:
        for a in sorted(set(ni.ALPHAS[cid]) | ({1e-2} if cid in (0, 1, 2, 3) else set()), reverse=True):
            cfg = ni.CONFIGS[cid].replace(alpha=a)
            W = ni.weights_trained(cfg)
            if W is None:
                continue
            f = ni.operator_factors(cfg)
            H = hierarchy(cfg, f, W)
            t0 = time.time()
            if cid == 0:
                y, _ = ni.make_rhs(cfg, f, a)
            elif cfg.dim == 1:
                y, _ = ni.make_rhs(cfg, f, a)
                y = y[IDX_1D]
            else:
                y, _ = ni.make_rhs(cfg, f, a, nrhs=2 if cid >= 3 else 4, start=0)
            orc = O.solve(H, y, tol=1e-6, max_cycles=150)
            key = f"{cfg.name}_a{a:g}"
            out[f"hist_{key}"] = orc.history
            out[f"cycles_{key}"] = orc.cycles
            out[f"conv_{key}"] = orc.converged
            print(f"{key}: converged {orc.converged.sum()}/{len(orc.converged)}, cycles {orc.cycles.max()} "
                  f"({time.time() - t0:.0f} s)", flush=True)
    np.savez_compressed(os.path.join(GOLD, "oracle_wtrain.npz"), **out)


def two_d():
    out = {}
    for key, (cid, a, m) in POOL_2D.items():
        cfg = ni.CONFIGS[cid].replace(alpha=a)
        f = ni.operator_factors(cfg)
        H = hierarchy(cfg, f, ni.weights_seed(cfg))
        pool, _ = ni.make_rhs(cfg, f, a, nrhs=8, start=0)
        t0 = time.time()
        orc = O.solve(H, pool[:m], tol=1e-300, max_cycles=3, freeze=False)
        out[f"hist_{key}"] = orc.history
        print(f"{key}: {m} RHS x 3 cycles in {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(os.path.join(GOLD, "oracle_2d_pool.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["1d_seed", "1d_lin", "2d"]
    for w in which:
        t0 = time.time()
        if w.startswith("trained:"):        # trained:0,1 -> only those configs (merged)
            trained(tuple(int(c) for c in w.split(":")[1].split(",")))
            continue
        {"1d_seed": one_d_seed, "1d_lin": one_d_lin, "2d": two_d, "trained": trained}[w]()
        print(f"{w} done in {time.time() - t0:.0f} s", flush=True)
