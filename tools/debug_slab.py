#!/usr/bin/env python
"""Dev tool: slab-sharded path (emulated ranks) vs the unsharded GPU path, step by step
variants (residual only; W_zero weights = pure coarse correction; filter off; full)."""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import nmg_inputs as ni  # noqa: E402


def main():
    import torch
    import paper_2603_01064_b200 as nmg
    from paper_2603_01064_b200.parallel import join_slabs, split_slabs
    dev = torch.device("cuda:0")
    cfg = ni.CONFIGS[2].replace(n=int(sys.argv[1]) if len(sys.argv) > 1 else 256, levels=5, nrhs=2)
    f = ni.operator_factors(cfg)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)

    def unsharded(W, filt, nu1, nu2):
        h = nmg.Hierarchy(2, cfg.n, cfg.levels, cfg.alpha, f, nu1=nu1, nu2=nu2, level_filter=filt, max_rhs=2)
        for l, w in enumerate(W):
            h.load_weights(l + 1, ni.cnn_arch(cfg), w)
        yd = torch.tensor(y, dtype=torch.float64, device=dev)
        xd = torch.zeros_like(yd)
        h.vcycle(yd, xd)
        r = torch.zeros_like(yd)
        rr = torch.zeros(2, dtype=torch.float64, device=dev)
        h.residual(yd, xd, r, rr)
        torch.cuda.synchronize()
        return xd.cpu().numpy(), rr.cpu().numpy()

    def sharded(world, W, filt, nu1, nu2):
        comms = nmg.Comm.emulated(world)
        ys = split_slabs(y, cfg.n, world)
        out = [None] * world
        errs = []

        def rk(r):
            try:
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    h = nmg.Hierarchy(2, cfg.n, cfg.levels, cfg.alpha, f, nu1=nu1, nu2=nu2, level_filter=filt,
                                      max_rhs=2, comm=comms[r])
                    for l, w in enumerate(W):
                        h.load_weights(l + 1, ni.cnn_arch(cfg), w)
                    yd = torch.tensor(np.ascontiguousarray(ys[r]), dtype=torch.float64, device=dev)
                    xd = torch.zeros_like(yd)
                    h.vcycle(yd, xd)
                    rr = torch.zeros(2, dtype=torch.float64, device=dev)
                    h.residual(yd, xd, None, rr)
                    torch.cuda.synchronize()
                    out[r] = (xd.cpu().numpy(), rr.cpu().numpy())
                    h.close()
            except Exception as e:  # noqa: BLE001
                errs.append(e)
        ts = [threading.Thread(target=rk, args=(r,)) for r in range(world)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        [c.close() for c in comms]
        if errs:
            raise errs[0]
        return join_slabs([o[0] for o in out], cfg.n), out[0][1]

    for wname in ("zero", "seed"):
        W = ni.weights_zero(cfg) if wname == "zero" else ni.weights_seed(cfg)
        for filt in (False, True):
            for nu1, nu2 in ((0, 0), (1, 0), (1, 1)):
                xa, ra = unsharded(W, filt, nu1, nu2)
                for world in (1, 2, 4):
                    try:
                        xb, rb = sharded(world, W, filt, nu1, nu2)
                        xa = xa.reshape(xb.shape)
                        d = np.linalg.norm(xa - xb) / max(np.linalg.norm(xa), 1e-300)
                        print(f"W={wname:4s} filt={int(filt)} nu=({nu1},{nu2}) world={world}: x rel diff {d:.3e}  "
                              f"relres {ra} vs {rb}", flush=True)
                    except Exception as e:  # noqa: BLE001
                        print(f"W={wname} filt={int(filt)} nu=({nu1},{nu2}) world={world}: ERROR {e}", flush=True)


if __name__ == "__main__":
    main()
