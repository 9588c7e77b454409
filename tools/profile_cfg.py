#!/usr/bin/env python
"""Per-kernel-class device times of one NMGF step for a BASELINE config (dev tool).

Usage: python tools/profile_cfg.py CFG [NRHS] [STEPS]
RHS are a seeded pool of 8 distinct right-hand sides tiled to NRHS (throughput does
not depend on the values).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nmg_inputs as ni  # noqa: E402


def main():
    import torch
    import paper_2603_01064_b200 as nmg
    cid = int(sys.argv[1])
    cfg = ni.CONFIGS[cid]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.nrhs
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    f = ni.operator_factors(cfg)
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, f, nu1=cfg.nu1, nu2=cfg.nu2, max_rhs=B)
    for l, w in enumerate(ni.weights_seed(cfg)):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    pool, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=min(8, B))
    reps = -(-B // pool.shape[0])
    y = torch.tensor(np.concatenate([pool] * reps)[:B], dtype=torch.float64, device="cuda")
    x = torch.zeros_like(y)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    h.vcycle(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h.vcycle(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    h.profile(True)
    for _ in range(steps):
        h.vcycle(y, x)
    torch.cuda.synchronize()
    h.profile(False)
    q = h.profile_query()
    print(f"cfg{cid} n={cfg.n} L={cfg.levels} B={B}: {ms:.3f} ms/step, {B / ms * 1e3:.1f} RHS*cycles/s")
    for k, (t, c) in q.items():
        print(f"   {k:9s} {t / steps:9.3f} ms/step  {c / steps:6.1f} launches/step")


if __name__ == "__main__":
    main()
