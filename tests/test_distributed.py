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


# ---------------------------------------------------------------- slab-sharded mode (config 4)
def _slab_worker(rank, world, port, out_dir):
    """Host model of the slab decomposition the library runs per rank (nmg_api.cu apply_slab /
    smooth_slab): Kronecker apply with one all-gather of the intermediate, CNN on the slab plus
    4 halo rows (zero padding only at the global image border), level filter with all-to-all
    transposes.  Each piece is compared with the unsharded oracle operator."""
    import torch
    import torch.distributed as dist

    import nmg_inputs as ni
    from oracle import nmg_oracle as O
    from paper_2603_01064_b200.parallel import slab_rows, split_slabs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = ni.CONFIGS[4].replace(n=32, levels=2, nrhs=2, sigma=0.08, channels=4)
    f = ni.operator_factors(cfg)
    H = O.build_hierarchy(2, f, cfg.alpha, cfg.levels)
    for l, w in enumerate(ni.weights_seed(cfg)):
        O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    n = cfg.n
    r0, R = slab_rows(n, world, rank)
    X = np.random.default_rng(3).standard_normal((2, n, n))      # row-major [i2][i1] images
    Xs = split_slabs(X, n, world)[rank]
    Bm, Cm = f                                                    # G = B (x) C: A X = C X B^T + alpha X

    # apply: T = (X[slab] C^T) local, all-gather, own output rows = B[slab] T_full + alpha X[slab]
    T = np.einsum("bij,kj->bik", Xs, Cm)                          # [b][i2 in slab][i1]
    parts = [torch.zeros(2, R, n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(T))
    Tf = np.concatenate([p.numpy() for p in parts], axis=1)       # [b][i2][i1]
    Ys = np.einsum("ij,bjk->bik", Bm[r0:r0 + R], Tf) + cfg.alpha * Xs
    want = O.apply_A(H, 0, X)[:, r0:r0 + R]
    apply_err = float(np.abs(Ys - want).max() / np.abs(want).max())

    # CNN: slab + 4 halo rows from the neighbours, zero padding only at the global border
    hal = [torch.zeros(2, n, n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(hal, torch.from_numpy(np.ascontiguousarray(X)))   # (a real run sends 4 rows)
    lo, hi = max(0, r0 - 4), min(n, r0 + R + 4)
    ext = hal[rank].numpy()[:, lo:hi]
    out = O.cnn_forward(H.weights[0], ext)[:, r0 - lo:r0 - lo + R]
    cnn_err = float(np.abs(out - O.cnn_forward(H.weights[0], X)[:, r0:r0 + R]).max())

    # level filter: row DFTs local, all-to-all transpose, column DFT x mask x inverse, back
    Z = np.fft.fft(Xs, axis=2)                                    # [b][rows][k1]
    cw = n // world
    send = [torch.from_numpy(np.ascontiguousarray(Z[:, :, d * cw:(d + 1) * cw])) for d in range(world)]
    recv = [torch.zeros(2, R, cw, dtype=torch.complex128) for _ in range(world)]
    dist.all_to_all(recv, send) if dist.get_backend() != "gloo" else _a2a_gloo(dist, send, recv, rank, world)
    col = np.concatenate([r.numpy() for r in recv], axis=1)       # [b][i2][k1 in my columns]
    a = lambda k: 2 * np.minimum(k, n - k) / n                     # noqa: E731  (reading R5)
    k1 = np.arange(rank * cw, (rank + 1) * cw)
    m = np.sqrt(np.maximum(a(np.arange(n))[:, None], a(k1)[None, :]))
    col = np.fft.ifft(np.fft.fft(col, axis=1) * m, axis=1)
    back = [torch.from_numpy(np.ascontiguousarray(col[:, q * R:(q + 1) * R])) for q in range(world)]
    got = [torch.zeros(2, R, cw, dtype=torch.complex128) for _ in range(world)]
    _a2a_gloo(dist, back, got, rank, world)
    Zs = np.concatenate([g.numpy() for g in got], axis=2)
    filt = np.real(np.fft.ifft(Zs, axis=2))
    filt_err = float(np.abs(filt - O.level_filter(H, 0, X)[:, r0:r0 + R]).max())
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), np.array([apply_err, cnn_err, filt_err]))
    dist.destroy_process_group()


def _a2a_gloo(dist, send, recv, rank, world):
    """all-to-all from point-to-point sends (gloo has no all_to_all)."""
    reqs = []
    for q in range(world):
        if q == rank:
            recv[q].copy_(send[q])
            continue
        reqs.append(dist.isend(send[q], q))
        reqs.append(dist.irecv(recv[q], q))
    for r in reqs:
        r.wait()


def test_slab_decomposition_gloo(tmp_path):
    world = 2
    mp.spawn(_slab_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        apply_err, cnn_err, filt_err = np.load(tmp_path / f"slab{r}.npy")
        assert apply_err < 1e-13 and cnn_err < 1e-13 and filt_err < 1e-13, (r, apply_err, cnn_err, filt_err)


def test_slab_rows_and_split_join():
    from paper_2603_01064_b200.parallel import join_slabs, slab_rows, split_slabs
    assert [slab_rows(1024, 8, r) for r in (0, 7)] == [(0, 128), (896, 128)]
    with pytest.raises(ValueError):
        slab_rows(100, 8, 0)
    y = np.arange(3 * 64.0).reshape(3, 64)
    s = split_slabs(y, 8, 4)
    assert all(p.shape == (3, 2, 8) and p.flags["C_CONTIGUOUS"] for p in s)
    assert np.array_equal(join_slabs(s, 8), y)
