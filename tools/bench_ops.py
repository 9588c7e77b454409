#!/usr/bin/env python
"""Time single level operations via the debug entry (dev tool).

Usage: python tools/bench_ops.py CONFIG OP[,OP...] [LEVEL...]
  OP in apply, residual, restrict, prolong, filter, cnn, smooth, coarse; levels are 1-based
  (coarse runs at level L regardless).
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nmg_inputs as ni

OPS = ("apply", "residual", "restrict", "prolong", "filter", "cnn", "smooth", "coarse")


def main():
    import torch
    import paper_2603_01064_b200 as nmg
    cid = int(sys.argv[1])
    ops = sys.argv[2].split(",")
    cfg = ni.CONFIGS[cid]
    B = min(cfg.nrhs, int(os.environ.get("NMG_OPS_RHS", cfg.nrhs)))
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, ni.operator_factors(cfg), nu1=cfg.nu1,
                      nu2=cfg.nu2, max_rhs=B)
    for l, w in enumerate(ni.weights_seed(cfg)):
        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    levels = [int(v) for v in sys.argv[3:]] or list(range(1, cfg.levels + 1))
    for name in ops:
        op = OPS.index(name)
        for lvl in ([cfg.levels] if name == "coarse" else levels):
            n = cfg.n >> (lvl - 1)
            shp = (B, n) if cfg.dim == 1 else (B, n, n)
            if name == "restrict":
                shp_out = shp[:1] + tuple(v // 2 for v in shp[1:])
            elif name == "prolong":
                shp, shp_out = shp[:1] + tuple(v // 2 for v in shp[1:]), shp
            else:
                shp_out = shp
            if name == "restrict" and lvl == cfg.levels:
                continue
            if name == "prolong" and lvl == cfg.levels:
                continue
            inp = torch.randn(*shp, device="cuda")
            out = torch.zeros(*shp_out, device="cuda")
            h.debug_op(lvl, op, inp, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record()
            for _ in range(reps):
                h.debug_op(lvl, op, inp, out)
            e1.record()
            torch.cuda.synchronize()
            print(f"cfg{cid} B={B} level {lvl} n={n} {name:8s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us")


if __name__ == "__main__":
    main()
