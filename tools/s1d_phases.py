#!/usr/bin/env python
"""Dev tool: 1D smoother class time per step with the level filter on / off and nu variants
(cfg 1 workload), to split the smoother's time between the CNN pipeline and the FFT filter."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nmg_inputs as ni  # noqa: E402


def run(filt, B=1024, steps=10):
    import torch
    import paper_2603_01064_b200 as nmg
    cfg = ni.CONFIGS[1]
    f = ni.operator_factors(cfg)
    h = nmg.Hierarchy(1, cfg.n, cfg.levels, cfg.alpha, f, nu1=1, nu2=1, level_filter=filt, max_rhs=B)
    for l, w in enumerate(ni.weights_seed(cfg)):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    y = torch.tensor(ni.make_rhs(cfg, f, cfg.alpha, nrhs=B)[0], dtype=torch.float64, device="cuda")
    x = torch.zeros_like(y)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for _ in range(3):
        h.vcycle(y, x)
    torch.cuda.synchronize()
    h.profile(True)
    for _ in range(steps):
        h.vcycle(y, x)
    torch.cuda.synchronize()
    h.profile(False)
    q = h.profile_query()
    print(f"filter={filt}: " + "  ".join(f"{k} {v[0] / steps:.3f}" for k, v in q.items()))


if __name__ == "__main__":
    run(True)
    run(False)
