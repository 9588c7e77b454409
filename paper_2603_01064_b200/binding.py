"""ctypes binding of include/nmg.h (argument marshalling only; every step of the
path runs in libnmg.so).  Device buffers are torch CUDA tensors (plumbing);
host buffers are numpy arrays or CPU tensors.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# NMG_LIB: alternative build of the same library (dev experiments with compile-time variants)
lib_path = os.environ.get("NMG_LIB") or os.path.join(HERE, "libnmg.so")

OP_APPLY, OP_RESIDUAL, OP_RESTRICT, OP_PROLONG, OP_FILTER, OP_CNN, OP_SMOOTH, OP_COARSE, OP_CYCLE0 = range(9)

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "SHAPE", 3: "NOT_SPD", 4: "NO_WEIGHTS", 5: "NONFINITE",
          6: "CUDA", 7: "OOM", 8: "UNSUPPORTED", 9: "DIVERGED", 10: "NCCL"}
PREC_MIXED, PREC_FP64 = 0, 1

EXPORTS = ["nmg_create_hierarchy", "nmg_load_smoother_weights", "nmg_vcycle", "nmg_solve",
           "nmg_vcycles_host", "nmg_residual", "nmg_debug_level_op", "nmg_launch_count",
           "nmg_destroy_hierarchy", "nmg_last_error", "nmg_version", "nmg_profile", "nmg_profile_query",
           "nmg_comm_nccl_unique_id", "nmg_comm_create_nccl", "nmg_comm_create_emulated", "nmg_comm_destroy",
           "nmg_create_hierarchy_slab", "nmg_load_fno_weights"]

KERNEL_CLASSES = ["gemm64", "gemm32", "smooth", "transfer", "coarse", "misc", "filter"]


class NmgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"nmg status {STATUS.get(status, status)}: {msg}")
        self.status = status


class Tuning(C.Structure):
    """nmg_tuning: kernel-selection knobs, all 0 = the default production path."""
    _fields_ = [("lanes", C.c_int32), ("no_graphs", C.c_int32), ("coarse_subst", C.c_int32),
                ("fp64_dmma", C.c_int32), ("simt_gemm", C.c_int32), ("ffma_cnn", C.c_int32),
                ("no_kron", C.c_int32), ("host_chunks", C.c_int32), ("fused_coarse", C.c_int32),
                ("no_compaction", C.c_int32), ("dense_k", C.c_int32),
                ("no_balance", C.c_int32), ("simt_fno", C.c_int32)]


class ProblemDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32), ("levels", C.c_int32), ("alpha", C.c_double),
                ("nu1", C.c_int32), ("nu2", C.c_int32), ("level_filter", C.c_int32),
                ("max_rhs", C.c_int32), ("device", C.c_int32), ("precision", C.c_int32),
                ("divergence_check", C.c_int32), ("tuning", C.POINTER(Tuning))]


class CnnArch(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("channels", C.c_int32), ("ksize", C.c_int32)]


class FnoArch(C.Structure):
    _fields_ = [("width", C.c_int32), ("n_layers", C.c_int32), ("modes", C.c_int32), ("ksize", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("cycles", C.POINTER(C.c_int32)), ("converged", C.POINTER(C.c_uint8)),
                ("history", C.POINTER(C.c_double)), ("wall_seconds", C.c_double),
                ("total_cycles", C.c_int32), ("fail_cycle", C.c_int32), ("fail_rhs", C.c_int32)]


_LIB = None


def load_library(path: Optional[str] = None):
    """Load libnmg.so; raises if it is missing (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = path or lib_path
    if not os.path.exists(p):
        raise ImportError(f"libnmg.so not built at {p}; run paper_2603_01064_b200/build.py "
                          "(there is no CPU fallback)")
    lib = C.CDLL(p)
    vp, i32, f64 = C.c_void_p, C.c_int32, C.c_double
    lib.nmg_create_hierarchy.argtypes = [C.POINTER(ProblemDesc), vp, C.POINTER(vp)]
    lib.nmg_load_smoother_weights.argtypes = [vp, i32, C.POINTER(CnnArch), vp, C.c_size_t]
    lib.nmg_load_fno_weights.argtypes = [vp, i32, C.POINTER(FnoArch), vp, C.c_size_t]
    lib.nmg_vcycle.argtypes = [vp, i32, vp, vp, vp]
    lib.nmg_solve.argtypes = [vp, i32, vp, vp, f64, i32, C.POINTER(Report), vp]
    lib.nmg_vcycles_host.argtypes = [vp, i32, vp, vp, i32, vp, vp]
    lib.nmg_residual.argtypes = [vp, i32, vp, vp, vp, vp, vp]
    lib.nmg_debug_level_op.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    lib.nmg_profile.argtypes = [vp, i32]
    lib.nmg_profile.restype = C.c_int
    lib.nmg_profile_query.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    lib.nmg_profile_query.restype = C.c_int
    lib.nmg_launch_count.argtypes = [vp]
    lib.nmg_launch_count.restype = C.c_int64
    lib.nmg_destroy_hierarchy.argtypes = [vp]
    lib.nmg_destroy_hierarchy.restype = None
    lib.nmg_last_error.restype = C.c_char_p
    lib.nmg_version.restype = C.c_char_p
    lib.nmg_comm_nccl_unique_id.argtypes = [vp]
    lib.nmg_comm_create_nccl.argtypes = [i32, i32, vp, i32, C.POINTER(vp)]
    lib.nmg_comm_create_emulated.argtypes = [i32, C.POINTER(vp)]
    lib.nmg_comm_destroy.argtypes = [vp]
    lib.nmg_comm_destroy.restype = None
    lib.nmg_create_hierarchy_slab.argtypes = [C.POINTER(ProblemDesc), vp, vp, C.POINTER(vp)]
    for f in ("nmg_create_hierarchy", "nmg_load_smoother_weights", "nmg_load_fno_weights", "nmg_vcycle", "nmg_solve",
              "nmg_vcycles_host", "nmg_residual", "nmg_debug_level_op", "nmg_comm_nccl_unique_id",
              "nmg_comm_create_nccl", "nmg_comm_create_emulated", "nmg_create_hierarchy_slab"):
        getattr(lib, f).restype = C.c_int
    _LIB = lib
    return lib


def _check(st: int):
    if st != 0:
        raise NmgError(st, _LIB.nmg_last_error().decode())


def _ptr(t) -> int:
    """Raw pointer of a torch tensor (device or host) or numpy array."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    assert t.is_contiguous()
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (nmg_comm_nccl_unique_id), to broadcast from rank 0."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    _check(lib.nmg_comm_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


class Comm:
    """One rank's communicator of the slab-sharded mode (nmg_comm)."""

    def __init__(self, handle, world: int, rank: int, keep=None):
        self._c, self.world, self.rank, self._keep = handle, world, rank, keep

    @classmethod
    def nccl(cls, world: int, rank: int, uid: bytes, device: int = 0) -> "Comm":
        lib = load_library()
        c = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _check(lib.nmg_comm_create_nccl(world, rank, C.cast(buf, C.c_void_p), device, C.byref(c)))
        return cls(c, world, rank)

    @classmethod
    def emulated(cls, world: int) -> list:
        """`world` ranks in this process on one device; drive each from its own thread."""
        lib = load_library()
        arr = (C.c_void_p * world)()
        _check(lib.nmg_comm_create_emulated(world, arr))
        return [cls(C.c_void_p(arr[r]), world, r) for r in range(world)]

    def close(self):
        if getattr(self, "_c", None):
            _LIB.nmg_comm_destroy(self._c)
            self._c = None


class Hierarchy:
    """Owns an nmg_hierarchy handle (C ABI nmg_create_hierarchy ... nmg_destroy_hierarchy).
    With `comm`, the handle is this rank's part of a slab-sharded 2D hierarchy
    (nmg_create_hierarchy_slab): vectors are the rank's slab [nrhs][n / world][n]."""

    def __init__(self, dim: int, n: int, levels: int, alpha: float, factors: Sequence[np.ndarray],
                 nu1: int = 1, nu2: int = 1, level_filter: bool = True, max_rhs: int = 1,
                 device: int = 0, comm: Optional[Comm] = None, precision: int = PREC_MIXED,
                 divergence_check: bool = False, tuning: Optional[dict] = None):
        lib = load_library()
        tun = Tuning(**(tuning or {}))
        d = ProblemDesc(dim, n, levels, float(alpha), nu1, nu2, int(level_filter), max_rhs, device,
                        int(precision), int(divergence_check), C.pointer(tun))
        fac = np.ascontiguousarray(np.concatenate([np.asarray(f, np.float64).ravel() for f in factors]))
        h = C.c_void_p()
        if comm is None:
            _check(lib.nmg_create_hierarchy(C.byref(d), fac.ctypes.data, C.byref(h)))
        else:
            _check(lib.nmg_create_hierarchy_slab(C.byref(d), fac.ctypes.data, comm._c, C.byref(h)))
        self._h = h
        self.comm = comm
        self.dim, self.n, self.levels, self.alpha = dim, n, levels, alpha
        self.max_rhs = max_rhs
        self.N = n if dim == 1 else n * n

    def close(self):
        if getattr(self, "_h", None):
            _LIB.nmg_destroy_hierarchy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_weights(self, level: int, arch, params: np.ndarray):
        p = np.ascontiguousarray(params, dtype=np.float32)
        a = CnnArch(*arch)
        _check(_LIB.nmg_load_smoother_weights(self._h, level, C.byref(a), p.ctypes.data, p.size))

    def load_fno_weights(self, level: int, arch, params: np.ndarray):
        """arch = (width, n_layers, modes, ksize); params flat fp32 (nmg_inputs.fno_param_shapes)."""
        p = np.ascontiguousarray(params, dtype=np.float32)
        a = FnoArch(*arch)
        _check(_LIB.nmg_load_fno_weights(self._h, level, C.byref(a), p.ctypes.data, p.size))

    def vcycle(self, y, x, stream=None):
        _check(_LIB.nmg_vcycle(self._h, y.shape[0], _ptr(y), _ptr(x), _stream(stream)))

    def residual(self, y, x, r=None, relres=None, stream=None):
        _check(_LIB.nmg_residual(self._h, y.shape[0], _ptr(y), _ptr(x), _ptr(r), _ptr(relres), _stream(stream)))

    def solve(self, y, x, tol: float = 1e-6, max_cycles: int = 50, stream=None):
        nrhs = y.shape[0]
        cyc = np.zeros(nrhs, np.int32)
        conv = np.zeros(nrhs, np.uint8)
        hist = np.full((nrhs, max_cycles + 1), np.nan)
        rep = Report(cyc.ctypes.data_as(C.POINTER(C.c_int32)), conv.ctypes.data_as(C.POINTER(C.c_uint8)),
                     hist.ctypes.data_as(C.POINTER(C.c_double)), 0.0, 0, -1, -1)
        st = _LIB.nmg_solve(self._h, nrhs, _ptr(y), _ptr(x), float(tol), int(max_cycles), C.byref(rep),
                            _stream(stream))
        out = dict(cycles=cyc, converged=conv.astype(bool), history=hist, wall_seconds=rep.wall_seconds,
                   total_cycles=rep.total_cycles, fail_cycle=rep.fail_cycle, fail_rhs=rep.fail_rhs, status=st)
        if st != 0:
            err = NmgError(st, _LIB.nmg_last_error().decode())
            err.report = out
            raise err
        return out

    def vcycles_host(self, y_host: np.ndarray, x_host: np.ndarray, cycles: int, relres: Optional[np.ndarray] = None,
                     stream=None):
        _check(_LIB.nmg_vcycles_host(self._h, y_host.shape[0], _ptr(y_host), _ptr(x_host), int(cycles),
                                     _ptr(relres), _stream(stream)))

    def debug_op(self, level: int, op: int, inp, out, stream=None):
        _check(_LIB.nmg_debug_level_op(self._h, level, op, inp.shape[0], _ptr(inp), _ptr(out), _stream(stream)))

    def profile(self, enable: bool):
        _check(_LIB.nmg_profile(self._h, int(enable)))

    def profile_query(self) -> dict:
        """{class: (total_ms, launches)} for the events recorded while profiling."""
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            ms, cnt = C.c_double(), C.c_int64()
            _check(_LIB.nmg_profile_query(self._h, i, C.byref(ms), C.byref(cnt)))
            out[name] = (ms.value, cnt.value)
        return out

    def launch_count(self) -> int:
        return int(_LIB.nmg_launch_count(self._h))


def version() -> str:
    return load_library().nmg_version().decode()
