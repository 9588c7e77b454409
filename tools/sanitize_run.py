#!/usr/bin/env python
"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): config 0,
a 2D 64x64 three-level hierarchy (tensor-core conv + Kronecker GEMMs), every debug op."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nmg_inputs as ni

def run(cfg, nrhs):
    import torch
    import paper_2603_01064_b200 as nmg
    f = ni.operator_factors(cfg)
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, f, nu1=cfg.nu1, nu2=cfg.nu2, max_rhs=nrhs)
    for l, w in enumerate(ni.weights_seed(cfg)):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=nrhs)
    yd = torch.tensor(y, dtype=torch.float64, device="cuda")
    xd = torch.zeros_like(yd)
    rep = h.solve(yd, xd, tol=1e-300, max_cycles=2)
    shp = (nrhs,) + (cfg.n,) * cfg.dim
    b = torch.randn(shp, device="cuda")
    for op in (nmg.OP_APPLY, nmg.OP_RESIDUAL, nmg.OP_FILTER, nmg.OP_CNN, nmg.OP_SMOOTH, nmg.OP_CYCLE0):
        h.debug_op(1, op, b, torch.zeros_like(b))
    torch.cuda.synchronize()
    print(cfg.name, "history", rep["history"][:, -1])

def run_fno(cfg, nrhs):
    """FNO smoothers (tcgen05 W-convolution: box kernel, and the row-halo kernel at 2D n >= 128)."""
    import torch
    import paper_2603_01064_b200 as nmg
    f = ni.operator_factors(cfg)
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, f, nu1=cfg.nu1, nu2=cfg.nu2, max_rhs=nrhs)
    for l, w in enumerate(ni.fno_weights_seed(cfg, seed=3)):
        h.load_fno_weights(l + 1, ni.fno_arch(cfg.dim, cfg.n >> l), w)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=nrhs)
    yd = torch.tensor(y, dtype=torch.float64, device="cuda")
    rep = h.solve(yd, torch.zeros_like(yd), tol=1e-300, max_cycles=1)
    torch.cuda.synchronize()
    print(cfg.name, "fno history", rep["history"][:, -1])


if __name__ == "__main__":
    if "fno" in sys.argv[1:]:
        run_fno(ni.CONFIGS[0].replace(nrhs=2), 2)
        run_fno(ni.CONFIGS[2].replace(n=128, levels=4, nrhs=1), 1)
        sys.exit(0)
    run(ni.CONFIGS[0], 8)
    run(ni.CONFIGS[2].replace(n=64, levels=3), 3)
    print("sanitize run done")
