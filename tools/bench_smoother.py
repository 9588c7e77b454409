#!/usr/bin/env python
"""Time the 1D smoother variants via the debug entry (dev tool): CNN only vs full smoothing step."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nmg_inputs as ni

def main():
    import torch
    import paper_2603_01064_b200 as nmg
    cfg = ni.CONFIGS[1]
    f = ni.operator_factors(cfg)
    h = nmg.Hierarchy(1, cfg.n, cfg.levels, cfg.alpha, f, max_rhs=1024)
    for l, w in enumerate(ni.weights_seed(cfg)):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    for lvl in (1, 2, 3, 4, 5):
        n = cfg.n >> (lvl - 1)
        b = torch.randn(1024, n, device="cuda")
        x = torch.zeros_like(b)
        for op, name in ((nmg.OP_CNN, "cnn"), (nmg.OP_SMOOTH, "smooth"), (nmg.OP_FILTER, "filter")):
            h.debug_op(lvl, op, b, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                h.debug_op(lvl, op, b, x)
            e1.record()
            torch.cuda.synchronize()
            print(f"level {lvl} n={n} {name:7s} {e0.elapsed_time(e1) / 10:.3f} ms")

if __name__ == "__main__":
    main()
