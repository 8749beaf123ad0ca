"""Thin ctypes binding of librtucker (include/rtucker.h).  Argument marshalling only:
every step of the method runs in the library's CUDA kernels.  PyTorch supplies device
memory, streams and (for NCCL bootstrap) process groups.

The library is loaded from this package directory; if it is missing the import fails
loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtucker.so")

MAX_MODES = 8
F32, F64 = 0, 1
DEVICE, HOST = 0, 1

STRICT = 1 << 0
ACCUM_AUTO = 0 << 1
ACCUM_FP64 = 1 << 1
ACCUM_FAST = 2 << 1
ACCUM_HYBRID = 3 << 1
ADAPT_NO_TRUNCATE = 1 << 3
ADAPT_HOSVD = 1 << 4
RESULT_HOST = 1 << 5
NO_CORE = 1 << 6
DETERMINISTIC = 1 << 7
DEBUG_CHECKS = 1 << 8
SP_HOSVD = 1 << 9
GRAPH = 1 << 10
EXACT_SVD = 1 << 16


def POWER(q: int) -> int:
    """RTUCKER_POWER(q): q steps of randomized subspace iteration."""
    return (int(q) & 15) << 12



ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)

STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ENUMERIC", 4: "ECUDA", 5: "ENCCL", 6: "EUNSUPPORTED"}

EXPORTED = [
    "rtucker_ctx_create", "rtucker_ctx_destroy", "rtucker_ctx_set_stream", "rtucker_last_error",
    "rtucker_launch_count", "rtucker_nccl_unique_id", "rtucker_version", "rtucker_hosvd", "rtucker_sthosvd",
    "rtucker_adaptive", "rtucker_sparse_sthosvd", "rtucker_result_free", "rtucker_memcpy", "rtucker_sync",
    "rtucker_rel_error", "rtucker_debug_sketch", "rtucker_debug_omega", "rtucker_debug_philox",
    "rtucker_debug_qr", "rtucker_debug_eig", "rtucker_debug_srrqr", "rtucker_set_profiling",
    "rtucker_phase_times", "rtucker_debug_gram_eig", "rtucker_debug_ttm", "rtucker_debug_loopback_sharding",
    "rtucker_debug_gemm", "rtucker_debug_gram", "rtucker_debug_coo_sketch", "rtucker_debug_gram_eig_ex",
]
PHASES = ("sketch", "qr", "bpass", "eig", "shrink", "other")


class RTuckerError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class DenseDesc(C.Structure):
    _fields_ = [("dtype", C.c_int), ("d", C.c_int32), ("dims", C.c_int64 * MAX_MODES),
                ("shard_offset", C.c_int64), ("shard_extent", C.c_int64), ("memory", C.c_int),
                ("data", C.c_void_p)]


class CooDesc(C.Structure):
    _fields_ = [("dtype", C.c_int), ("d", C.c_int32), ("dims", C.c_int64 * MAX_MODES), ("nnz", C.c_int64),
                ("memory", C.c_int), ("idx", C.c_void_p * MAX_MODES), ("vals", C.c_void_p)]


class ResultStruct(C.Structure):
    _fields_ = [("d", C.c_int32), ("dims", C.c_int64 * MAX_MODES), ("ranks", C.c_int64 * MAX_MODES),
                ("ell", C.c_int64 * MAX_MODES), ("order", C.c_int32 * MAX_MODES), ("seed", C.c_uint64),
                ("flags", C.c_uint32), ("dtype", C.c_int), ("memory", C.c_int), ("core", C.c_void_p),
                ("factors", C.c_void_p * MAX_MODES), ("mode_residual_sq", C.c_double * MAX_MODES),
                ("norm_sq", C.c_double), ("core_nnz", C.c_int64), ("core_idx", C.c_void_p * MAX_MODES),
                ("core_vals", C.c_void_p), ("selection", C.c_void_p * MAX_MODES),
                ("nnz_history", C.c_int64 * (MAX_MODES + 1)), ("swaps", C.c_int32 * MAX_MODES),
                ("internal", C.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load librtucker.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"librtucker.so not found at {path}; run `python -m paper_1905_07311_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    P, I32, I64, U32, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    RP = C.POINTER(C.POINTER(ResultStruct))
    sig = {
        "rtucker_ctx_create": (C.c_int, [C.c_int, P, P, C.c_int, C.c_int, ALLOC_FN, FREE_FN, P, C.POINTER(P)]),
        "rtucker_ctx_destroy": (None, [P]),
        "rtucker_ctx_set_stream": (C.c_int, [P, P]),
        "rtucker_last_error": (C.c_char_p, [P]),
        "rtucker_launch_count": (U64, [P]),
        "rtucker_nccl_unique_id": (C.c_int, [P]),
        "rtucker_version": (C.c_char_p, []),
        "rtucker_hosvd": (C.c_int, [P, C.POINTER(DenseDesc), P, I32, U64, U32, RP]),
        "rtucker_sthosvd": (C.c_int, [P, C.POINTER(DenseDesc), P, I32, U64, P, U32, RP]),
        "rtucker_adaptive": (C.c_int, [P, C.POINTER(DenseDesc), D, I32, P, P, U64, U32, RP]),
        "rtucker_sparse_sthosvd": (C.c_int, [P, C.POINTER(CooDesc), P, I32, U64, P, D, U32, RP]),
        "rtucker_result_free": (None, [P, C.POINTER(ResultStruct)]),
        "rtucker_memcpy": (C.c_int, [P, P, P, C.c_size_t, C.c_int]),
        "rtucker_sync": (C.c_int, [P]),
        "rtucker_rel_error": (C.c_int, [P, C.POINTER(DenseDesc), C.POINTER(ResultStruct), C.POINTER(D)]),
        "rtucker_debug_sketch": (C.c_int, [P, C.POINTER(DenseDesc), I32, I32, I64, U64, U32, P]),
        "rtucker_debug_omega": (C.c_int, [P, C.c_int, U64, I32, P, I64, I32, I64, P]),
        "rtucker_debug_philox": (C.c_int, [P, P, I64, U32, U32, P]),
        "rtucker_debug_qr": (C.c_int, [P, I64, I32, P, P]),
        "rtucker_debug_eig": (C.c_int, [P, I32, P, P, P, C.POINTER(I32)]),
        "rtucker_debug_srrqr": (C.c_int, [P, I64, I32, P, D, P, P, C.POINTER(I32)]),
        "rtucker_debug_coo_sketch": (C.c_int, [P, C.POINTER(CooDesc), I32, I32, U64, U32, P]),
        "rtucker_debug_gram_eig": (C.c_int, [P, I32, P, P, P, C.POINTER(I32)]),
        "rtucker_debug_gram_eig_ex": (C.c_int, [P, I32, P, P, P, C.POINTER(I32), I32, I32]),
        "rtucker_debug_ttm": (C.c_int, [P, C.POINTER(DenseDesc), I32, P, I32, U32, P, P]),
        "rtucker_debug_loopback_sharding": (C.c_int, [P, C.c_int]),
        "rtucker_set_profiling": (C.c_int, [P, C.c_int]),
        "rtucker_debug_gemm": (C.c_int, [P, C.c_int, C.c_int, I64, I64, I64, P, I64, P, I64, P, I64]),
        "rtucker_debug_gram": (C.c_int, [P, I64, I64, I64, P, P]),
        "rtucker_phase_times": (C.c_int, [P, P, P, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


# ----------------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _dtype_code(dt) -> int:
    s = str(dt)
    if "float64" in s or s in ("f64", "double"):
        return F64
    if "float32" in s or s in ("f32", "float"):
        return F32
    raise TypeError(f"unsupported dtype {dt} (float32 / float64 only)")


def _buffer(x):
    """(pointer, memory, dtype code, keepalive) for a torch tensor or numpy array."""
    try:
        torch = _torch()
        if isinstance(x, torch.Tensor):
            if not x.is_contiguous():
                raise ValueError("tensor must be contiguous (first-mode-fastest memory image)")
            mem = DEVICE if x.is_cuda else HOST
            return x.data_ptr(), mem, _dtype_code(x.dtype), x
    except ImportError:
        pass
    a = np.ascontiguousarray(x) if not (isinstance(x, np.ndarray) and (x.flags.c_contiguous or x.flags.f_contiguous)) else x
    return a.ctypes.data, HOST, _dtype_code(a.dtype), a


@dataclass
class TuckerResult:
    core: np.ndarray | None
    factors: list
    ranks: tuple
    ell: tuple
    order: tuple
    seed: int
    mode_residual_sq: tuple
    norm_sq: float
    # sparse
    core_idx: np.ndarray | None = None
    core_vals: np.ndarray | None = None
    selections: list = field(default_factory=list)
    nnz_history: tuple = ()
    swaps: tuple = ()


class Result:
    """Owns an rtucker_result*.  `numpy()` copies a host result into numpy arrays."""

    def __init__(self, ctx: "Context", ptr):
        self.ctx = ctx
        self.ptr = ptr

    @property
    def s(self) -> ResultStruct:
        return self.ptr.contents

    def free(self):
        if self.ptr:
            self.ctx.lib.rtucker_result_free(self.ctx.h, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def numpy(self) -> TuckerResult:
        s = self.s
        d = s.d
        ranks = tuple(int(s.ranks[k]) for k in range(d))
        dims = tuple(int(s.dims[k]) for k in range(d))
        host = s.memory == HOST

        def grab(ptr, n, ctype, npdt):
            if not ptr or n == 0:
                return np.zeros(0, dtype=npdt)
            if host:
                return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).copy()
            out = np.empty(n, dtype=npdt)
            self.ctx._check(self.ctx.lib.rtucker_memcpy(self.ctx.h, out.ctypes.data, ptr, out.nbytes, 2))
            self.ctx.sync()
            return out

        vt, vdt = (C.c_double, np.float64) if s.dtype == F64 else (C.c_float, np.float32)
        core = None
        if s.core:
            core = grab(s.core, int(np.prod(ranks)), C.c_double, np.float64).reshape(ranks, order="F")
        factors = []
        for k in range(d):
            if s.factors[k]:
                factors.append(grab(s.factors[k], dims[k] * ranks[k], C.c_double, np.float64)
                               .reshape((dims[k], ranks[k]), order="F"))
            else:
                factors.append(None)
        out = TuckerResult(core, factors, ranks, tuple(int(s.ell[k]) for k in range(d)),
                           tuple(int(s.order[k]) for k in range(d)), int(s.seed),
                           tuple(float(s.mode_residual_sq[k]) for k in range(d)), float(s.norm_sq))
        if s.core_nnz or s.core_vals:
            nnz = int(s.core_nnz)
            out.core_idx = np.stack([grab(s.core_idx[k], nnz, C.c_int32, np.int32) for k in range(d)])
            out.core_vals = grab(s.core_vals, nnz, vt, vdt)
            out.selections = [grab(s.selection[k], ranks[k], C.c_int64, np.int64) for k in range(d)]
            out.nnz_history = tuple(int(s.nnz_history[k]) for k in range(d + 1))
            out.swaps = tuple(int(s.swaps[k]) for k in range(d))
        return out


class Context:
    """One library context per GPU / rank.

    device: CUDA ordinal; stream: a torch.cuda.Stream (default: torch's current stream);
    group: optional torch.distributed process group for the multi-rank (NCCL) path;
    allocator: "library" (default) uses the library's own stream-ordered pool; "torch" routes
    the library's device workspace and results through torch's caching allocator
    (rtucker_alloc_fn hooks: memory shared with torch, at ~50 us of host time per allocation
    for the Python callback -- 5.6 ms/step of host enqueue on eager C4 calls against 0.25 ms
    with the pool)."""

    def __init__(self, device: int = 0, stream=None, group=None, rank: int | None = None,
                 world: int | None = None, nccl_id: bytes | None = None, allocator: str = "library"):
        self.lib = load_library()
        torch = _torch()
        if stream is None and torch.cuda.is_available():
            stream = torch.cuda.current_stream(device)
            if stream.cuda_stream == 0:  # legacy default stream: give the library a real one
                stream = torch.cuda.Stream(device)
        self.stream = stream
        sp = C.c_void_p(stream.cuda_stream) if stream is not None else None
        idbuf = None
        r, n = 0, 1
        if group is not None or (world or 1) > 1:
            import torch.distributed as dist
            r = dist.get_rank(group) if rank is None else rank
            n = dist.get_world_size(group) if world is None else world
            if n > 1:
                if nccl_id is None:
                    nccl_id = bootstrap_nccl_id(group, r)
                idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        h = C.c_void_p()
        self._alloc_cb, self._free_cb = ALLOC_FN(), FREE_FN()   # NULL hooks: library pool
        if allocator == "torch":
            self._alloc_cb, self._free_cb = _torch_hooks(device)
        elif allocator != "library":
            raise ValueError("allocator must be 'torch' or 'library'")
        st = self.lib.rtucker_ctx_create(device, sp, idbuf, r, n, self._alloc_cb, self._free_cb, None, C.byref(h))
        if st != 0:
            raise RTuckerError(st, "rtucker_ctx_create failed")
        self.h = h
        self.rank, self.world = r, n

    def close(self):
        if getattr(self, "h", None):
            self.lib.rtucker_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise RTuckerError(st, self.lib.rtucker_last_error(self.h).decode())

    def _enter(self):
        """Order the library stream after the work already queued on torch's current stream
        (inputs produced there)."""
        if self.stream is not None:
            torch = _torch()
            cur = torch.cuda.current_stream(self.stream.device)
            if cur.cuda_stream != self.stream.cuda_stream:
                self.stream.wait_stream(cur)

    @property
    def launches(self) -> int:
        return int(self.lib.rtucker_launch_count(self.h))

    def sync(self):
        self._check(self.lib.rtucker_sync(self.h))

    def loopback_sharding(self, on: bool = True):
        self._check(self.lib.rtucker_debug_loopback_sharding(self.h, 1 if on else 0))

    def set_profiling(self, on: bool = True):
        self._check(self.lib.rtucker_set_profiling(self.h, 1 if on else 0))

    def phase_times(self, reset: bool = True):
        """{(phase, position): (total_ms, count)} from the library's CUDA events."""
        ms = (C.c_double * (6 * MAX_MODES))()
        n = (C.c_int64 * (6 * MAX_MODES))()
        self._check(self.lib.rtucker_phase_times(self.h, ms, n, 1 if reset else 0))
        out = {}
        for ph in range(6):
            for pos in range(MAX_MODES):
                k = ph * MAX_MODES + pos
                if n[k]:
                    out[(PHASES[ph], pos)] = (float(ms[k]), int(n[k]))
        return out

    # ------------------------------------------------------------------ descriptors
    def dense_desc(self, x, dims, shard=None):
        """x: a flat first-mode-fastest memory image (1-D torch tensor or numpy array), or
        a logical-shape numpy array (converted with Fortran-order ravel).  Also orders the
        library stream after torch's current stream (where x may have been produced)."""
        self._enter()
        if isinstance(x, np.ndarray) and x.ndim > 1:
            x = np.ravel(x, order="F")
        elif hasattr(x, "dim") and x.dim() > 1:
            raise ValueError("pass torch tensors as flat first-mode-fastest images")
        ptr, mem, dt, keep = _buffer(x)
        dims = [int(v) for v in dims]
        d = DenseDesc()
        d.dtype, d.d, d.memory, d.data = dt, len(dims), mem, ptr
        for k, v in enumerate(dims[:MAX_MODES]):   # d > 8 is rejected by the library
            d.dims[k] = v
        if shard is not None:
            d.shard_offset, d.shard_extent = int(shard[0]), int(shard[1])
        return d, keep

    @staticmethod
    def _i64(v):
        a = (C.c_int64 * max(1, len(v)))(*[int(t) for t in v])
        return a

    @staticmethod
    def _i32(v):
        return None if v is None else (C.c_int32 * len(v))(*[int(t) for t in v])

    # ------------------------------------------------------------------- algorithms
    def sthosvd(self, x, dims, ranks, p, seed=0, order=None, flags=0, shard=None) -> Result:
        """R-STHOSVD (Alg 3).  x: first-mode-fastest tensor (torch CUDA/CPU or numpy)."""
        desc, keep = self.dense_desc(x, dims, shard)
        out = C.POINTER(ResultStruct)()
        self._check(self.lib.rtucker_sthosvd(self.h, C.byref(desc), self._i64(ranks), int(p), int(seed),
                                             self._i32(order), int(flags), C.byref(out)))
        del keep
        return Result(self, out)

    def hosvd(self, x, dims, ranks, p, seed=0, flags=0, shard=None) -> Result:
        """R-HOSVD (Alg 2)."""
        desc, keep = self.dense_desc(x, dims, shard)
        out = C.POINTER(ResultStruct)()
        self._check(self.lib.rtucker_hosvd(self.h, C.byref(desc), self._i64(ranks), int(p), int(seed),
                                           int(flags), C.byref(out)))
        return Result(self, out)

    def adaptive(self, x, dims, tol, block, mode_tol=None, order=None, seed=0, flags=0, shard=None) -> Result:
        """Adaptive R-STHOSVD (Alg 5); flags ADAPT_HOSVD selects Alg 4."""
        desc, keep = self.dense_desc(x, dims, shard)
        out = C.POINTER(ResultStruct)()
        mt = None if mode_tol is None else (C.c_double * len(mode_tol))(*[float(t) for t in mode_tol])
        self._check(self.lib.rtucker_adaptive(self.h, C.byref(desc), float(tol), int(block), mt,
                                              self._i32(order), int(seed), int(flags), C.byref(out)))
        return Result(self, out)

    def _coo_desc(self, idx, vals, dims):
        d = len(dims)
        desc = CooDesc()
        keep = []
        vptr, mem, dt, kv = _buffer(vals)
        keep.append(kv)
        desc.dtype, desc.d, desc.memory, desc.vals = dt, d, mem, vptr
        for k in range(d):
            desc.dims[k] = int(dims[k])
            row = idx[k]
            iptr, imem, _, ki = _buffer_int32(row)
            if imem != mem:
                raise ValueError("indices and values must live in the same memory")
            desc.idx[k] = iptr
            keep.append(ki)
        desc.nnz = int(len(vals))
        return desc, keep

    def sparse_sthosvd(self, idx, vals, dims, ranks, p, seed=0, order=None, eta=2.0, flags=0) -> Result:
        """SP-STHOSVD (Alg 6).  idx: (d, nnz) int32 (torch or numpy, 0-based); vals: values."""
        desc, keep = self._coo_desc(idx, vals, dims)
        self._enter()
        out = C.POINTER(ResultStruct)()
        self._check(self.lib.rtucker_sparse_sthosvd(self.h, C.byref(desc), self._i64(ranks), int(p), int(seed),
                                                    self._i32(order), float(eta), int(flags), C.byref(out)))
        return Result(self, out)

    def rel_error(self, x, dims, res: Result) -> float:
        desc, keep = self.dense_desc(x, dims)
        v = C.c_double()
        self._check(self.lib.rtucker_rel_error(self.h, C.byref(desc), res.ptr, C.byref(v)))
        return v.value

    # ----------------------------------------------------------------------- debug
    def debug_sketch(self, x, dims, mode, ell, seed=0, k0=0, flags=0):
        torch = _torch()
        desc, keep = self.dense_desc(x, dims)
        y = torch.empty(int(ell) * int(dims[mode]), dtype=torch.float64, device="cuda")
        self._check(self.lib.rtucker_debug_sketch(self.h, C.byref(desc), int(mode), int(ell), int(k0), int(seed),
                                                  int(flags), y.data_ptr()))
        self.sync()
        return y.cpu().numpy().reshape((int(dims[mode]), int(ell)), order="F")

    def debug_coo_sketch(self, idx, vals, dims, mode, ell, seed=0, flags=0):
        """Y = X_(mode) Omega_mode[:, :ell] of a COO tensor (Alg 6 line 4), fp64 (I_mode x ell)."""
        torch = _torch()
        desc, keep = self._coo_desc(idx, vals, dims)
        y = torch.empty(int(ell) * int(dims[mode]), dtype=torch.float64, device="cuda")
        self._check(self.lib.rtucker_debug_coo_sketch(self.h, C.byref(desc), int(mode), int(ell), int(seed),
                                                      int(flags), y.data_ptr()))
        self.sync()
        return y.cpu().numpy().reshape((int(dims[mode]), int(ell)), order="F")

    def debug_ttm(self, x, dims, mode, a, flags=0, want_out=True, want_gram=True):
        """B = A^T X_(mode) as (L, J, R) fp64 and its Gram (J x J)."""
        torch = _torch()
        desc, keep = self.dense_desc(x, dims)
        at = torch.as_tensor(np.asfortranarray(a, dtype=np.float64).ravel(order="F"), device="cuda")
        J = a.shape[1]
        L = int(np.prod(dims[:mode], dtype=np.int64))
        R = int(np.prod(dims[mode + 1:], dtype=np.int64))
        out = torch.empty(L * J * R, dtype=torch.float64, device="cuda") if want_out else None
        g = torch.empty(J * J, dtype=torch.float64, device="cuda") if want_gram else None
        self._check(self.lib.rtucker_debug_ttm(self.h, C.byref(desc), int(mode), at.data_ptr(), int(J), int(flags),
                                               out.data_ptr() if out is not None else None,
                                               g.data_ptr() if g is not None else None))
        self.sync()
        return (out, g.cpu().numpy().reshape((J, J), order="F") if g is not None else None)

    def debug_omega(self, cols, ell, seed=0, mode=0, k0=0, dtype="f64"):
        torch = _torch()
        cols_t = torch.as_tensor(np.asarray(cols, dtype=np.int64), device="cuda")
        tdt = torch.float64 if dtype == "f64" else torch.float32
        out = torch.empty(int(ell) * cols_t.numel(), dtype=tdt, device="cuda")
        self._check(self.lib.rtucker_debug_omega(self.h, F64 if dtype == "f64" else F32, int(seed), int(mode),
                                                 cols_t.data_ptr(), cols_t.numel(), int(ell), int(k0),
                                                 out.data_ptr()))
        self.sync()
        return out.cpu().numpy().reshape((cols_t.numel(), int(ell)), order="F")

    def debug_philox(self, ctr: np.ndarray, key0: int, key1: int):
        torch = _torch()
        c = torch.as_tensor(np.asarray(ctr, dtype=np.uint32).view(np.int32).ravel(), device="cuda")
        out = torch.empty_like(c)
        self._check(self.lib.rtucker_debug_philox(self.h, c.data_ptr(), c.numel() // 4, int(key0), int(key1),
                                                  out.data_ptr()))
        self.sync()
        return out.cpu().numpy().view(np.uint32).reshape(-1, 4)

    def debug_qr(self, y: np.ndarray):
        torch = _torch()
        m, n = y.shape
        yt = torch.as_tensor(np.asfortranarray(y, dtype=np.float64).ravel(order="F"), device="cuda")
        q = torch.empty_like(yt)
        self._check(self.lib.rtucker_debug_qr(self.h, m, n, yt.data_ptr(), q.data_ptr()))
        self.sync()
        return q.cpu().numpy().reshape((m, n), order="F")

    def debug_eig(self, a: np.ndarray):
        torch = _torch()
        n = a.shape[0]
        at = torch.as_tensor(np.asfortranarray(a, dtype=np.float64).ravel(order="F"), device="cuda")
        w = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty_like(at)
        sw = C.c_int32()
        self._enter()
        self._check(self.lib.rtucker_debug_eig(self.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw)))
        self.sync()
        self.last_sweeps = int(sw.value)
        return w.cpu().numpy(), v.cpu().numpy().reshape((n, n), order="F")

    def debug_gram_eig(self, a: np.ndarray):
        """Hot-path PSD eigensolver (pivoted Cholesky + one-sided Jacobi)."""
        torch = _torch()
        n = a.shape[0]
        at = torch.as_tensor(np.asfortranarray(a, dtype=np.float64).ravel(order="F"), device="cuda")
        w = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty_like(at)
        sw = C.c_int32()
        self._enter()
        self._check(self.lib.rtucker_debug_gram_eig(self.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(), C.byref(sw)))
        self.sync()
        self.last_sweeps = int(sw.value)
        return w.cpu().numpy(), v.cpu().numpy().reshape((n, n), order="F")

    def debug_gram_eig_ex(self, a: np.ndarray, rel_acc: bool, r_need: int):
        """The hot path's Gram eigensolver as selected for fp32 (rel_acc False) / fp64 data."""
        torch = _torch()
        n = a.shape[0]
        at = torch.as_tensor(np.asfortranarray(a, dtype=np.float64).ravel(order="F"), device="cuda")
        w = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty_like(at)
        sw = C.c_int32()
        self._enter()
        self._check(self.lib.rtucker_debug_gram_eig_ex(self.h, n, at.data_ptr(), w.data_ptr(), v.data_ptr(),
                                                       C.byref(sw), int(bool(rel_acc)), int(r_need)))
        self.sync()
        self.last_sweeps = int(sw.value)
        return w.cpu().numpy(), v.cpu().numpy().reshape((n, n), order="F")

    def debug_gemm(self, a: np.ndarray, b: np.ndarray, transA=False, transB=False):
        """C = op(A) op(B) through the library's fp64 tensor-core GEMM."""
        torch = _torch()
        at = torch.as_tensor(np.asfortranarray(a, dtype=np.float64).ravel(order="F"), device="cuda")
        bt = torch.as_tensor(np.asfortranarray(b, dtype=np.float64).ravel(order="F"), device="cuda")
        m = a.shape[1] if transA else a.shape[0]
        k = a.shape[0] if transA else a.shape[1]
        n = b.shape[0] if transB else b.shape[1]
        c = torch.empty(m * n, dtype=torch.float64, device="cuda")
        self._enter()
        self._check(self.lib.rtucker_debug_gemm(self.h, int(transA), int(transB), m, n, k, at.data_ptr(), a.shape[0],
                                                bt.data_ptr(), b.shape[0], c.data_ptr(), m))
        self.sync()
        return c.cpu().numpy().reshape((m, n), order="F")

    def debug_gram(self, b: np.ndarray, L: int, K: int, R: int):
        """Gram of the mode unfolding of an fp64 tensor stored (L, K, R) (flat image b)."""
        torch = _torch()
        bt = torch.as_tensor(np.asarray(b, dtype=np.float64).ravel(), device="cuda")
        c = torch.empty(K * K, dtype=torch.float64, device="cuda")
        self._enter()
        self._check(self.lib.rtucker_debug_gram(self.h, L, K, R, bt.data_ptr(), c.data_ptr()))
        self.sync()
        return c.cpu().numpy().reshape((K, K), order="F")

    def debug_srrqr(self, q: np.ndarray, eta: float = 2.0):
        torch = _torch()
        m, l = q.shape
        qt = torch.as_tensor(np.asfortranarray(q, dtype=np.float64).ravel(order="F"), device="cuda")
        sel = torch.empty(l, dtype=torch.int64, device="cuda")
        a = torch.empty_like(qt)
        sw = C.c_int32()
        self._check(self.lib.rtucker_debug_srrqr(self.h, m, l, qt.data_ptr(), float(eta), sel.data_ptr(),
                                                 a.data_ptr(), C.byref(sw)))
        self.sync()
        return sel.cpu().numpy(), a.cpu().numpy().reshape((m, l), order="F"), int(sw.value)


def _torch_hooks(device: int):
    """rtucker_alloc_fn / rtucker_free_fn routed to torch's caching allocator (stream-ordered
    on the library's stream, so freed blocks are reused in stream order)."""
    torch = _torch()

    def _alloc(nbytes, stream, user):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0)))
        except Exception:  # out of memory or any allocator error: NULL -> RTUCKER_ENOMEM
            return None

    def _free(ptr, stream, user):
        if ptr:
            torch.cuda.caching_allocator_delete(int(ptr))

    return ALLOC_FN(_alloc), FREE_FN(_free)


def _buffer_int32(x):
    try:
        torch = _torch()
        if isinstance(x, torch.Tensor):
            if x.dtype != torch.int32 or not x.is_contiguous():
                raise TypeError("COO indices must be contiguous int32")
            return x.data_ptr(), (DEVICE if x.is_cuda else HOST), None, x
    except ImportError:
        pass
    a = np.ascontiguousarray(x, dtype=np.int32)
    return a.ctypes.data, HOST, None, a


def bootstrap_nccl_id(group, rank: int) -> bytes:
    """Rank 0 creates a ncclUniqueId and broadcasts it over the torch process group."""
    import torch
    import torch.distributed as dist
    lib = load_library()
    buf = C.create_string_buffer(128)
    if rank == 0:
        st = lib.rtucker_nccl_unique_id(buf)
        if st != 0:
            raise RTuckerError(st, "ncclGetUniqueId failed")
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).to(dev)
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().numpy().tobytes())
