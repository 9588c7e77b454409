#!/usr/bin/env python
"""Benchmark of the batched NMGF solve phase (arxiv 2603.01064) on B200.

Default workload (--config 3): BASELINE.json configs[3], the largest configuration that fits
one GPU -- 2D 512 x 512, sigma = 0.02, alpha = 1e-3 (--alpha 1e-4 for the other sweep point),
6 levels (512^2 -> 16^2), 2048 RHS sharded over the ranks, CNN 4 x 48 3x3 smoothers (W_seed),
nu1 = nu2 = 1, level filter on.  --config 0..4 selects the other BASELINE rows.

One "step" = one pass of the whole hot path over the batch: fp64 outer residual and
convergence test, one NMGF V-cycle (all levels), fp64 update.
  value = RHS * V-cycles / s, whole job (all ranks), device-timed (CUDA events, max over
          ranks).  Configs 1-4 split the configuration's own RHS batch over the ranks
          (strong scaling); config 0 runs replicas; config 4 row-shards its
          single operator (slab mode) over NCCL.
  e2e   = the same metric through the C ABI host-buffer entry nmg_vcycles_host (H2D of y
          and x from pinned host memory, one cycle, D2H of x inside the timed region),
          checked afterwards against the device entry.
  solve = RHS solved to 1e-6 relative residual per second with the converging W_lin
          stand-in weights (1D configs only).
Inputs are larger than L2 (cfg 3: 4 GiB fp64 y and x), so no explicit L2 flush is needed.

--smoother fno runs the same cycle with the paper's FNO smoothers (Table-6 architecture per level,
W_seed weights; W-convolutions as 3xTF32 implicit GEMMs on tcgen05) instead of BASELINE's CNNs;
its line reports the FNO smoother class against the 3xTF32 tensor peak and has no solve figure
(no trained FNO weights exist here).

--impl reference times the fp64 CPU oracle (oracle/) on a bounded sample of the same
workload on this host's cores (the reference arm: /root/reference holds only the paper).
"""
from __future__ import annotations

import argparse
import json
import math
import os
# NCCL's banner / debug lines (NCCL_DEBUG=VERSION in some images) go to stderr: stdout carries
# only the one JSON line per run
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import nmg_inputs as ni  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
FP64_NOMINAL_RATIO = 45.0 / 2250.0     # B200 nominal FP64 / dense BF16 (blackwell guide)
TF32_NOMINAL_RATIO = 1100.0 / 2250.0


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        p["source"] = "measured (MEASURED_PEAKS.json)"
        return p
    except Exception:
        p = dict(FALLBACK)
        p["source"] = "fallback (B200_PROFILING.md)"
        return p


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()                 # the sampler is running before the timed region starts
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic counts
def algorithmic_counts(cfg, B):
    """Per-step algorithmic FLOPs / bytes per kernel class."""
    n = [cfg.n >> l for l in range(cfg.levels)]
    L = cfg.levels
    if cfg.dim == 2:
        # Kronecker pair: 2 GEMMs of 2 n^3 FLOP per RHS per apply; applies per level:
        # pre residual + post residual (+ extra smoothing steps)
        g64 = 4.0 * B * n[0] ** 3
        g32 = sum(4.0 * B * n[l] ** 3 * (1 + cfg.nu2 + max(cfg.nu1 - 1, 0)) for l in range(L - 1))
        C = cfg.channels
        per_px = 2 * (9 * C + 2 * 9 * C * C + 9 * C)
        sm = sum((cfg.nu1 + cfg.nu2) * B * n[l] ** 2 * per_px for l in range(L - 1))
        return {"gemm64": g64, "gemm32": g32, "smooth": sm}
    g64 = 2.0 * B * n[0] * n[0]
    g32 = 0.0
    for l in range(L - 1):
        # r_l = y - A x (n x n), b_post = r - (A P) e (n x n/2)
        g32 += 2.0 * B * n[l] * n[l] * (1.0 + (0.5 if cfg.nu2 else 0.0))
        g32 += 2.0 * B * n[l] * n[l] * (max(cfg.nu1 - 1, 0) + max(cfg.nu2 - 1, 0))
    cnn_per_pt = 2 * (cfg.channels * cfg.ksize + cfg.channels * cfg.channels * cfg.ksize + cfg.channels * cfg.ksize)
    sm = sum((cfg.nu1 + cfg.nu2) * B * n[l] * cnn_per_pt for l in range(L - 1))
    return {"gemm64": g64, "gemm32": g32, "smooth": sm,
            "gemm64_bytes": 8.0 * (n[0] * n[0] + 3 * B * n[0])}


def fno_flops(cfg, B):
    """FNO smoother FLOPs per step (Appendix A / Table 6 arch per level): per Fourier layer the
    W-convolution 2 c^2 ks^d per point and the complex mode mixing 8 c^2 per kept mode (k in 1D,
    2k x k in 2D); lift and projection 2c per point each.  The FFTs of the kept modes are not
    counted."""
    tot = 0.0
    for l in range(cfg.levels - 1):
        n = cfg.n >> l
        c, L, k, ks = ni.fno_arch(cfg.dim, n)
        pts = n ** cfg.dim
        modes = k if cfg.dim == 1 else 2 * k * k
        tot += (cfg.nu1 + cfg.nu2) * B * (L * (2.0 * c * c * ks ** cfg.dim * pts + 8.0 * c * c * modes) + 4.0 * c * pts)
    return tot


# ------------------------------------------------------------------ oracle timing
def oracle_rate(cfg, factors, weights, y, nrhs, cycles, fno=False):
    from oracle import nmg_oracle as O
    H = O.build_hierarchy(cfg.dim, factors, cfg.alpha, cfg.levels, nu1=cfg.nu1, nu2=cfg.nu2)
    for l, w in enumerate(weights):
        if fno:
            O.load_weights(H, l + 1, O.fno_params(cfg.dim, *ni.fno_arch(cfg.dim, cfg.n >> l), w))
        else:
            O.load_weights(H, l + 1, ni.unflatten_params(cfg, w))
    ys = y[:nrhs]
    x = np.zeros_like(ys)
    t0 = time.perf_counter()
    for _ in range(cycles):
        x = O.nmgf_cycle(H, x, ys)
        O.relative_residual(H, x, ys)
    dt = time.perf_counter() - t0
    return nrhs * cycles / dt, dt


def host_threads():
    """Threads the oracle's numpy/BLAS actually uses on this host."""
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(th) if th else 1
    except Exception:
        return os.cpu_count()


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def metric_name(cfg):
    """Identical on both arms (the driver divides the two values)."""
    return f"RHS*V-cycles/s ({cfg.name})"


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--config", type=int, default=3, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--alpha", type=float, default=None, help="override the config's alpha (sweep points)")
    ap.add_argument("--nrhs", type=int, default=None)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--lanes", type=int, default=0, help="nmg_tuning.lanes (0 = library default, 1 = off)")
    ap.add_argument("--tune", default="", help="extra nmg_tuning fields, e.g. no_fused_coarse=1,no_graphs=1")
    ap.add_argument("--precision", choices=["auto", "mixed", "fp64"], default="auto",
                    help="auto: fp64 cycle for config 0 (BASELINE's fp64 system), mixed otherwise")
    ap.add_argument("--smoother", choices=["cnn", "fno"], default="cnn",
                    help="cnn: BASELINE's CNN smoothers (the headline); fno: the paper's FNO smoothers "
                         "(Table 6 hyperparameters per level, W_seed; W-convolutions on tcgen05, SURVEY NEXT-2)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--slab", choices=["auto", "on", "off"], default="auto",
                    help="config 4 at N > 1: row-shard the single operator over the ranks (SURVEY §8(e)); "
                         "auto = on for config 4 with N > 1 over NCCL")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cid = args.config
    cfg = ni.CONFIGS[cid]
    if args.alpha is not None:
        cfg = cfg.replace(alpha=args.alpha)
    if args.nrhs:
        cfg = cfg.replace(nrhs=args.nrhs)
    fno = args.smoother == "fno"
    if args.steps is None:
        args.steps = ({0: 500, 1: 10, 2: 3, 3: 1, 4: 2} if fno else
                      {0: 5000, 1: 400, 2: 60, 3: 5, 4: 30})[cid]   # >= ~0.5 s timed (clock samples)
    B = cfg.nrhs
    pool = cfg.dim == 2 and B > 8     # 2D: 8 seeded RHS tiled to the batch (throughput is value-independent)
    workload = (f"{cfg.name}_{cfg.dim}d_n{cfg.n}_L{cfg.levels}_rhs{B}"
                f"{'_per_gpu' if cid == 0 else '_total'}_alpha{cfg.alpha:g}_"
                f"{'FNO' if fno else 'C%d' % cfg.channels}_Wseed")

    def make_y(nrhs, start):
        if not pool:
            return ni.make_rhs(cfg, factors, cfg.alpha, nrhs=nrhs, start=start)[0]
        base = ni.make_rhs(cfg, factors, cfg.alpha, nrhs=8, start=start)[0]
        return np.ascontiguousarray(np.concatenate([base] * (-(-nrhs // 8)))[:nrhs])

    if args.impl == "reference":
        if rank != 0:
            return
        factors = ni.operator_factors(cfg)
        W = ni.fno_weights_seed(cfg, seed=3) if fno else ni.weights_seed(cfg)
        # bounded sample per step (every --steps / --warmup step runs): 1D 16 RHS x 1 cycle,
        # 2D 1 RHS x 1 cycle (cfg 3: ~3 s per step on 16 host threads)
        ns = 16 if cfg.dim == 1 else 1
        y, _ = ni.make_rhs(cfg, factors, cfg.alpha, nrhs=ns)
        secs = 0.0
        for _ in range(args.warmup):
            oracle_rate(cfg, factors, W, y, ns, 1, fno)
        for _ in range(args.steps):
            _, dt = oracle_rate(cfg, factors, W, y, ns, 1, fno)
            secs += dt
        v = args.steps * ns / secs
        sample = f"{ns} RHS x 1 cycle per step of the {cfg.name} workload"
        line = {"impl": "reference", "metric": metric_name(cfg), "value": v,
                "unit": "RHS*cycles/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
                "scaling": "weak" if cid == 0 else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "sample": sample},
                "cpu_baseline": {"value": v, "unit": "RHS*cycles/s", "cores": host_threads(), "kind": "oracle",
                                 "sample": sample, **host_info()},
                "e2e": {"value": v, "unit": "RHS*cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    import paper_2603_01064_b200 as nmg
    from paper_2603_01064_b200.parallel import max_over_ranks, shard_range, weak_shard

    if world > 1:
        ndev = torch.cuda.device_count()
        local = local % ndev            # (test mode only: more ranks than GPUs share devices)
        torch.cuda.set_device(local)
        backend = os.environ.get("NMG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    # configs 1-4: strong scaling -- the configuration's own RHS batch is split over the ranks
    # (RHS sharding needs no exchange step; config 4 at N > 1 row-shards its single
    # operator instead).  Config 0 (8 RHS, latency-bound) runs one replica per rank (weak).
    strong = cid != 0
    # config 4 over several GPUs: the single 1024^2 operator is row-sharded (slab mode, one
    # all-gather of the Kronecker intermediate per apply, all-to-all transposes in the level
    # filter); every rank holds its slab of all 32 RHS
    slab = (cfg.dim == 2 and args.slab == "on") or (
        args.slab == "auto" and cid == 4 and world > 1 and os.environ.get("NMG_DIST_BACKEND", "nccl") == "nccl")
    comm = None
    if slab:
        from paper_2603_01064_b200.parallel import split_slabs
        start, global_B = 0, cfg.nrhs
        obj = [nmg.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        comm = nmg.Comm.nccl(world, rank, obj[0], local)   # world 1: a one-rank NCCL communicator
    elif strong:
        start, B = shard_range(cfg.nrhs, world, rank)
        global_B = cfg.nrhs
    else:
        start, _ = weak_shard(B, rank)
        global_B = world * B
    factors = ni.operator_factors(cfg)
    W = ni.fno_weights_seed(cfg, seed=3) if fno else ni.weights_seed(cfg)
    if B == 0:
        raise SystemExit(f"rank {rank}: no RHS left for this rank ({cfg.nrhs} RHS over {world} ranks)")
    prec = nmg.PREC_FP64 if args.precision == "fp64" or (args.precision == "auto" and cid == 0 and not fno) else nmg.PREC_MIXED
    h = nmg.Hierarchy(cfg.dim, cfg.n, cfg.levels, cfg.alpha, factors, nu1=cfg.nu1, nu2=cfg.nu2, max_rhs=B,
                      device=local, comm=comm, precision=prec,
                      tuning={"lanes": args.lanes, **{k: int(v) for k, v in (kv.split("=") for kv in args.tune.split(",") if kv)}})
    for l, w in enumerate(W):
        if fno:
            h.load_fno_weights(l + 1, ni.fno_arch(cfg.dim, cfg.n >> l), w)
        else:
            h.load_weights(l + 1, ni.cnn_arch(cfg), w)
    y_np = make_y(B, start)
    if slab:
        y_np = np.ascontiguousarray(split_slabs(y_np, cfg.n, world)[rank])
    y = torch.tensor(y_np, dtype=torch.float64, device=dev)
    x = torch.zeros_like(y)
    stream = torch.cuda.Stream(dev)          # non-default stream: the library replays a CUDA graph
    torch.cuda.set_stream(stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        h.vcycle(y, x, stream)
    torch.cuda.synchronize(dev)

    # ---- timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = h.launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            h.vcycle(y, x, stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = h.launch_count() - l0
    ms = max_over_ranks(e0.elapsed_time(e1))
    value = global_B * args.steps / (ms / 1e3)

    # ---- per-kernel-class device times (CUDA events on the launching stream)
    psteps = min(args.steps, 100)                        # event pairs per launch: keep the pass short
    h.profile(True)
    for _ in range(psteps):
        h.vcycle(y, x, stream)
    torch.cuda.synchronize(dev)
    h.profile(False)
    prof = h.profile_query()
    tot_prof = sum(v[0] for v in prof.values())
    counts = algorithmic_counts(cfg, B)
    if fno:
        counts["smooth"] = fno_flops(cfg, B)
    pk = peaks()
    clocks = clk.summary()
    # the burst figure for a kernel timed alone, the sustained one for a kernel inside a long
    # step: a timed region that drove the GPU into its power cap is the condition the sustained
    # matmul figure was measured under (MEASURED_PEAKS.json "how")
    sustained = "sw_power_cap" in clocks["reasons"] and "bf16_tflops_sustained" in pk
    bf16_burst = pk["bf16_tflops"]
    bf16 = pk["bf16_tflops_sustained"] if sustained else bf16_burst
    dom = max(prof, key=lambda k: prof[k][0])
    dom_ms, dom_n = prof[dom]
    step_ms = dom_ms / psteps                           # all launches of the class in one step
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh).get(f"cfg{cid}", {}).get(dom)   # ncu dram read+write bytes per step
    except Exception:
        pass
    f16x3_peak = bf16 / 3.0      # f16 dense = bf16 dense rate; 3 products per fp32-accurate MAC
    if fno and dom == "smooth":
        # FNO smoother: the W-convolution (the dense contraction, > 95 % of the FNO FLOPs) runs as a
        # 3xTF32 implicit GEMM on tcgen05 (fno_tc.cu); the class also holds the mode FFTs, the mode
        # mixing, lift and projection (fp32 SIMT), so the fraction is a whole-smoother figure
        peak = bf16 * TF32_NOMINAL_RATIO / 3.0
        achieved = counts["smooth"] / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "fno_conv_rows_kernel / fno_conv_tc_kernel (W-conv + bias + GELU, 3xTF32 tcgen05 implicit "
                          "GEMM) + fno_* (lift, row/column mode FFTs, mode mixing, projection; fp32 SIMT), all "
                          "launches of a step",
                "bound": "tensor", "unit": "TFLOP/s",
                "peak_note": "TF32 tensor (measured bf16 x 1.1/2.25) / 3 products per fp32-accurate MAC; FNO FLOPs "
                             "= per layer 2 c^2 ks^d per point (W-conv) + 8 c^2 per kept mode (mixing), lift and "
                             "projection 2c; FFTs not counted"}
    elif dom == "gemm64":
        peak = bf16 * FP64_NOMINAL_RATIO
        achieved = counts["gemm64"] / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "fp64 outer residual (Ozaki int8 tcgen05 / DMMA)", "bound": "tensor", "unit": "TFLOP/s",
                "peak_note": "FP64 tensor: measured bf16 x nominal fp64/bf16 ratio 45/2250"}
    elif dom == "gemm32":
        peak = bf16 * TF32_NOMINAL_RATIO / 3.0
        achieved = counts["gemm32"] / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "tc_gemm_kernel (3xTF32 tcgen05, all levels)", "bound": "tensor", "unit": "TFLOP/s",
                "peak_note": "TF32 tensor (measured bf16 x 1.1/2.25) / 3 passes"}
    elif prec == nmg.PREC_FP64:
        # the whole cycle in one fused launch (cycle64_kernel, one CTA per RHS): latency-bound;
        # reported against the FP32 FFMA rate (148 SMs x 128 lanes x 2 FLOP x 1.965 GHz)
        peak = 148 * 128 * 2 * 1.965e9 / 1e12
        achieved = (counts["gemm64"] * 2 + counts["gemm32"] + counts["smooth"]) / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "cycle64_kernel (whole fp64 cycle per RHS, one CTA per RHS, one launch per cycle)",
                "bound": "alu", "unit": "TFLOP/s",
                "peak_note": "FP32 FFMA peak from unit counts and clock (DESIGN.md §6); work = fp64 operator "
                             "applies + fp32 CNN FLOPs; the kernel is latency-bound (8 CTAs on 148 SMs)"}
    elif cfg.dim == 1:
        peak = f16x3_peak
        achieved = counts["smooth"] / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "smooth1d_f16_kernel (norm, CNN with the 16->16 layer on tcgen05 FP16x3, level filter, "
                          "update), all launches of a step",
                "bound": "tensor", "unit": "TFLOP/s",
                "peak_note": "FP16 dense tensor = measured bf16 dense, / 3 products per fp32-accurate MAC; "
                             "CNN FLOPs (2880/point) only"}
    elif dom == "smooth":
        peak = f16x3_peak
        achieved = counts["smooth"] / (step_ms * 1e-3) / 1e12
        roof = {"kernel": "conv_strip_kernel<C,1> + <C,0> (2D CNN layers 1-2 / 3-4, FP16x3 tcgen05), all launches "
                          "of a step",
                "bound": "tensor", "unit": "TFLOP/s",
                "peak_note": "FP16 dense tensor = measured bf16 dense, / 3 products per fp32-accurate MAC; "
                             "CNN FLOPs (2 (9C + 18C^2 + 9C) per pixel) only"}
    else:
        peak = pk["hbm_gbs"] / 1e3
        achieved = (counts.get(dom + "_bytes") or float("nan")) / (step_ms * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "hbm", "unit": "TB/s"}
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": traffic,
                 "traffic_note": (f"ncu dram__bytes_read+write of the {dom} class per step (cfg{cid}), profiles/traffic.json"
                                  if traffic else None),
                 "peak_source": ("derived from unit counts and clock (DESIGN.md §6)" if roof["bound"] == "alu" else
                                 pk["source"] + (" bf16_tflops_sustained (run at sw_power_cap)" if sustained
                                                 else (" bf16_tflops (burst)" if roof["bound"] == "tensor"
                                                       else " hbm_gbs"))),
                 "frac_vs_burst_peak": (achieved / (peak * bf16_burst / bf16)) if roof["bound"] == "tensor" else None,
                 "share_of_step": dom_ms / tot_prof if tot_prof else None,
                 "classes_ms_per_step": {k: v[0] / psteps for k, v in prof.items()},
                 "launches_per_step": {k: v[1] / psteps for k, v in prof.items()}})

    # ---- end to end through the host-buffer C-ABI entry
    e2e = None
    if not args.no_e2e:
        yh = torch.empty(y.shape, dtype=torch.float64).pin_memory()
        xh = torch.zeros(y.shape, dtype=torch.float64).pin_memory()
        yh.copy_(torch.from_numpy(y_np))
        yhn, xhn = yh.numpy(), xh.numpy()
        def host_step():
            if not slab:
                h.vcycles_host(yhn, xhn, 1, stream=stream)
                return
            # slab mode: the rank's slab of y and x host -> device, one cycle, x device -> host
            y.copy_(yh, non_blocking=True)
            x.copy_(xh, non_blocking=True)
            h.vcycle(y, x, stream)
            xh.copy_(x, non_blocking=True)

        for _ in range(2):                                   # eager run, then graph capture
            host_step()
        barrier()
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            host_step()
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(f0.elapsed_time(f1))
        # correctness check of the path just timed: one host-entry cycle from x = 0 against one
        # device-entry cycle from x = 0 (same kernels; RHS chunking changes no per-RHS arithmetic)
        xh.zero_()
        host_step()
        torch.cuda.synchronize(dev)
        xd = torch.zeros_like(y)
        h.vcycle(y, xd, stream)
        torch.cuda.synchronize(dev)
        xdh = xd.cpu()
        diff = float((xh - xdh).abs().max() / xdh.abs().max().clamp_min(1e-300))
        e2e = {"value": global_B * args.steps / (ems / 1e3), "unit": "RHS*cycles/s",
               "h2d_bytes_per_step": 2 * 8 * B * cfg.N, "d2h_bytes_per_step": 8 * B * cfg.N,
               "check_vs_device_entry_max_rel_diff": diff}
        del yh, xh, xd

    # ---- RHS solved to 1e-6 / s with converging weights: the trained smoothers W_train
    # (trainer/nmg_train.py, Alg 5) for this config and alpha when present, else (1D) the W_lin
    # stand-in at the largest alpha of the sweep where it converges
    solve = None
    if not args.no_solve and not fno:      # no trained FNO weights exist
        wt = ni.weights_trained(cfg)
        scfg, label = cfg, "W_train (level-wise trainer, Alg 5)"
        if wt is None:            # the config's trained set at another alpha of the curriculum
            for a in (1e-2, 1e-3, 1e-4):
                if ni.weights_trained(cfg.replace(alpha=a)) is not None:
                    scfg = cfg.replace(alpha=a)
                    wt = ni.weights_trained(scfg)
                    break
        if wt is None and cfg.dim == 1:
            scfg = cfg.replace(alpha=max(ni.ALPHAS[cid]))
            wt, label = ni.weights_lin(scfg), "W_lin stand-in"
        if wt is not None:
            sf = ni.operator_factors(scfg)
            hs = nmg.Hierarchy(cfg.dim, scfg.n, scfg.levels, scfg.alpha, sf, nu1=scfg.nu1, nu2=scfg.nu2, max_rhs=B,
                               device=local, precision=prec)
            for l, w in enumerate(wt):
                hs.load_weights(l + 1, ni.cnn_arch(scfg), w)
            if scfg.alpha == cfg.alpha:
                ys = y
            else:
                ys = torch.tensor(make_y(B, start), dtype=torch.float64, device=dev)
            xs = torch.zeros_like(ys)
            hs.solve(ys, xs, tol=1e-6, max_cycles=100, stream=stream)   # warm (graph capture)
            xs.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            rep = hs.solve(ys, xs, tol=1e-6, max_cycles=100, stream=stream)
            sec = max_over_ranks(rep["wall_seconds"])
            conv = int(rep["converged"].sum())
            solve = {"value": (world if not strong else 1) * conv / sec * (world if strong else 1),
                     "unit": "RHS solved/s (relres<=1e-6)", "alpha": scfg.alpha, "weights": label,
                     "cycles_max": int(rep["cycles"].max()), "cycles_mean": float(rep["cycles"].mean()),
                     "converged": conv, "of": B, "seconds": sec}
            hs.close()
            del xs

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nr, nc = {0: (8, 200), 1: (128, 8), 2: (4, 2), 3: (1, 1), 4: (1, 1)}[cid]
        if fno:
            nr, nc = {0: (8, 20), 1: (16, 1), 2: (1, 1), 3: (1, 1), 4: (1, 1)}[cid]
        rate, dt = oracle_rate(cfg, factors, W, y_np, nr, nc, fno)
        cpu = {"value": rate, "unit": "RHS*cycles/s", "cores": host_threads(), "kind": "oracle",
               "sample": f"{nr} RHS x {nc} cycles of the same workload ({dt:.1f} s)", **host_info()}

    if rank == 0:
        line = {"metric": metric_name(cfg),
                "value": value, "unit": "RHS*cycles/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": ("f64 outer residual (Ozaki int8 tcgen05) + fp32-accurate inner cycle (FNO smoothers: 3xTF32 "
                          "tcgen05 W-convolutions, fp32 SIMT mode FFTs; tcgen05 operator applies)" if fno else
                          "f64 (NMG_PREC_FP64 fused cycle; the CNN's own arithmetic fp32)" if prec == nmg.PREC_FP64 else
                          "f64 outer residual (Ozaki int8 tcgen05) + fp32-accurate inner cycle (FP16x3 tcgen05 "
                          + ("CNN and operator applies)" if cfg.dim == 1 else "CNN, 3xTF32 tcgen05 Kronecker applies)")),
                "data": ("synthetic (seeded RHS; W_seed FNO weights, Table 6 arch per level)" if fno else
                         "synthetic (seeded RHS; W_seed Kaiming-uniform weights)"),
                "config": {"workload": workload, "global_batch": global_B, "n": cfg.n, "levels": cfg.levels,
                           "rhs": "8-RHS seeded pool tiled to the batch" if pool else "seeded, distinct",
                           "alpha": cfg.alpha, "nu1": cfg.nu1, "nu2": cfg.nu2,
                           "parallelism": (f"operator slab-shard x{world} (NCCL all-gather per apply)" if slab else
                                           f"rhs-shard x{world}" + (f" (strong: {cfg.nrhs} RHS split)" if strong
                                                                    else " (replicas)")),
                           "l2": ("working set fits L2 (latency-bound config, no flush)" if cid == 0
                                  else "inputs larger than L2 (no flush)")},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "solve": solve,
                "gpu_launches": launches, "clocks": clocks}
        print(json.dumps(line))
    if comm is not None:
        h.close()
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
