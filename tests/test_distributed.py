"""Multi-process (gloo, world_size 2, CPU) checks of the RHS-sharding host logic.

Each rank solves its RHS shard; the gathered per-RHS results must equal a single
process solving the whole batch (the NMGF cycle is per-RHS independent, so the
sharded path has no collective on the data path).  The compute here is the oracle
(CPU) -- the point is the shard/gather/timing plumbing that bench.py uses with the
CUDA path on GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_01064_b200.parallel import shard_range, weak_shard


def test_shard_range_covers_exactly():
    for total in (1, 7, 1024, 2048):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            idx = [i for s, c in spans for i in range(s, s + c)]
            assert idx == list(range(total))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    assert weak_shard(1024, 3) == (3072, 1024)
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import nmg_inputs as ni
    from oracle import nmg_oracle as O
    from paper_2603_01064_b200.parallel import gather_reports, max_over_ranks, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = ni.CONFIGS[0].replace(n=64, levels=3, nrhs=6)
    f = ni.operator_factors(cfg)
    H = O.build_hierarchy(1, f, cfg.alpha, cfg.levels)
    for l, w in enumerate(ni.weights_lin(cfg)):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    start, count = shard_range(cfg.nrhs, world, rank)
    y, _ = ni.make_rhs(cfg, f, cfg.alpha, nrhs=count, start=start)
    rep = O.solve(H, y, tol=1e-6, max_cycles=60)
    t = max_over_ranks(float(rank + 1))
    reports = gather_reports({"rank": rank, "start": start, "cycles": rep.cycles.tolist(),
                              "x": rep.x, "time": t})
    if rank == 0:
        np.save(os.path.join(out_dir, "x.npy"), np.concatenate([r["x"] for r in reports]))
        np.save(os.path.join(out_dir, "cycles.npy"), np.concatenate([r["cycles"] for r in reports]))
        np.save(os.path.join(out_dir, "time.npy"), np.array([r["time"] for r in reports]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import nmg_inputs as ni
    from oracle import nmg_oracle as O
    cfg = ni.CONFIGS[0].replace(n=64, levels=3, nrhs=6)
    f = ni.operator_factors(cfg)
    H = O.build_hierarchy(1, f, cfg.alpha, cfg.levels)
    for l, w in enumerate(ni.weights_lin(cfg)):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    y, _ = ni.make_rhs(cfg, f, cfg.alpha)
    rep = O.solve(H, y, tol=1e-6, max_cycles=60)
    xs = np.load(tmp_path / "x.npy")
    assert np.allclose(xs, rep.x, rtol=0, atol=1e-12 * np.abs(rep.x).max())
    assert np.array_equal(np.load(tmp_path / "cycles.npy"), rep.cycles)
    assert np.all(np.load(tmp_path / "time.npy") == 2.0)      # max over ranks
