"""Thin ctypes binding over libddks.so (include/ddks.h). Argument marshalling only: every step of the
hot path runs in the library's sm_100a kernels. There is no CPU fallback — if the extension is missing
this module raises at import, and on a machine without a GPU ddks_create returns DDKS_ERR_CUDA.

Inputs may be torch tensors (CUDA: read in place on the current torch stream; CPU: copied H2D inside the
library call, which is what the end-to-end measurement times) or NumPy arrays (host). Names mirror the C ABI.
"""
from __future__ import annotations

import ctypes
import os
import warnings
from typing import NamedTuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libddks.so")

DDKS_OK = 0
STATUS = {0: "DDKS_OK", 1: "DDKS_ERR_INVALID_ARGUMENT", 2: "DDKS_ERR_EMPTY_SAMPLE", 3: "DDKS_ERR_DIM_UNSUPPORTED",
          4: "DDKS_ERR_NONFINITE", 5: "DDKS_ERR_TOO_LARGE", 6: "DDKS_ERR_CUDA", 7: "DDKS_ERR_NCCL", 8: "DDKS_ERR_OOM"}
DDKS_FLAG_DEFAULT = 0
DDKS_FLAG_NO_VALIDATE = 1
DDKS_FLAG_TIES_GT = 2
DDKS_FLAG_FORCE_DIRECT = 4
DDKS_FLAG_PROFILE = 8
DDKS_FLAG_PERM_GATHER = 16
DDKS_FLAG_NO_X0 = 32
DDKS_FLAG_FORCE_X0 = 64
DDKS_FLAG_RDKS_FULL_SORT = 128
DDKS_FLAG_NO_RANK = 256
DDKS_FLAG_FORCE_RANK = 512
DDKS_FLAG_KD_SHIFT = 16
DDKS_FLAG_NCCL_SELF = 2048
DDKS_FLAG_NO_GRAPH = 4096


def DDKS_FLAG_KD_LEVELS(k: int) -> int:
    """TEST ONLY: force k (1..4) levels of kd ordering (include/ddks.h)."""
    return (k & 7) << DDKS_FLAG_KD_SHIFT
DDKS_SIG_POISSON = 1


class DDKSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ddks_result(ctypes.Structure):
    _fields_ = [("num", ctypes.c_uint64), ("den", ctypes.c_uint64), ("D", ctypes.c_double),
                ("argmax_origin", ctypes.c_int64)]


class ddks_rank_record(ctypes.Structure):
    _fields_ = [("num", ctypes.c_uint64), ("argmax_origin", ctypes.c_int64), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


class ddks_significance_result(ctypes.Structure):
    _fields_ = [("stat", ddks_result), ("S", ctypes.c_double), ("log_prod", ctypes.c_double), ("cells", ctypes.c_int64)]


class Significance(NamedTuple):
    stat: "Result"
    S: float
    log_prod: float
    cells: int
    mt_hist: np.ndarray | None
    log_p_table: np.ndarray | None


class Result(NamedTuple):
    num: int
    den: int
    D: float
    argmax_origin: int


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libddks.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is deliberately no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    sig = {
        "ddks_get_nccl_id": ([vp], ctypes.c_int),
        "ddks_create": ([ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, u32], ctypes.c_int),
        "ddks_stat": ([vp, vp, i64, vp, i64, i32, vp, ctypes.POINTER(ddks_result)], ctypes.c_int),
        "ddks_stat_batch": ([vp, vp, vp, i64, i64, i64, i32, vp, ctypes.POINTER(ddks_result)], ctypes.c_int),
        "ddks_permutation_null": ([vp, vp, i64, i64, i32, vp, i64, vp, vp, ctypes.POINTER(ddks_result),
                                   ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "ddks_stat_shard": ([vp, vp, i64, vp, i64, i32, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(ddks_result)],
                            ctypes.c_int),
        "ddks_stat_per_origin": ([vp, vp, i64, vp, i64, i32, i64, i64, vp, vp], ctypes.c_int),
        "ddks_significance": ([vp, vp, i64, vp, i64, i32, u32, vp, ctypes.POINTER(ddks_significance_result), vp, vp],
                              ctypes.c_int),
        "ddks_significance_batch": ([vp, vp, vp, i64, i64, i64, i32, u32, vp, vp], ctypes.c_int),
        "ddks_vdks": ([vp, vp, i64, vp, i64, i32, i64, vp, ctypes.POINTER(ddks_result)], ctypes.c_int),
        "ddks_rdks": ([vp, vp, i64, vp, i64, i32, vp, ctypes.POINTER(ddks_result)], ctypes.c_int),
        "ddks_shard_range": ([i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)], ctypes.c_int),
        "ddks_combine_records": ([ctypes.POINTER(ddks_rank_record), ctypes.c_int, ctypes.POINTER(ddks_rank_record)],
                                 ctypes.c_int),
        "ddks_unpad_items": ([vp, i64, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(u32)], ctypes.c_int),
        "ddks_profile_work": ([vp, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
        "ddks_launch_count": ([vp], i64),
        "ddks_kd_levels": ([vp], i32),
        "ddks_rank_lanes": ([vp], i32),
        "ddks_profile_clock": ([vp, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "ddks_profile_read": ([vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_uint64)],
                              ctypes.c_int),
        "ddks_destroy": ([vp], ctypes.c_int),
        "ddks_last_error": ([vp], ctypes.c_char_p),
        "ddks_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


LIB = _load()
EXPORTED = ("ddks_get_nccl_id", "ddks_create", "ddks_stat", "ddks_stat_batch", "ddks_permutation_null",
            "ddks_stat_per_origin", "ddks_stat_shard", "ddks_significance", "ddks_significance_batch", "ddks_vdks", "ddks_rdks", "ddks_shard_range", "ddks_combine_records", "ddks_unpad_items", "ddks_launch_count",
            "ddks_kd_levels", "ddks_rank_lanes", "ddks_profile_clock", "ddks_profile_read", "ddks_profile_work", "ddks_destroy",
            "ddks_last_error", "ddks_version")


def _check(st: int, ctx=None):
    if st != DDKS_OK:
        raise DDKSError(st, (LIB.ddks_last_error(ctx) or b"").decode())


try:  # torch is optional for the binding (NumPy inputs work without it); looked up once, not per call
    import torch as _torch
except ImportError:  # pragma: no cover
    _torch = None


def _torch_stream(stream):
    """The torch stream a call's conversions must run on: the caller's `stream` (a torch.cuda.Stream or a raw
    cudaStream_t handle), else torch's current stream."""
    import torch
    if stream is None:
        return torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream))


class _Arg:
    """Holds a pointer to a float32/int32 C-contiguous buffer (torch tensor or NumPy array) alive for a call.
    A CUDA tensor of another dtype or layout is converted ON THE CALL'S STREAM (the library reads it there), and a
    float64 input is cast to float32 with a warning: the library's coordinates are float32 (BASELINE.json configs), and
    the cast can merge distinct values into ties, which can change D relative to the float64 definition."""

    def __init__(self, x, dtype, stream=None):
        self.keep = None
        torch = _torch
        if torch is not None and isinstance(x, torch.Tensor):
            if dtype == np.float32 and x.dtype is torch.float32 and x.is_contiguous():  # the common case: as is
                self.keep = x
                self.ptr = x.data_ptr()
                self.shape = tuple(x.shape)
                self.is_cuda = x.is_cuda
                return
            tdt = torch.float32 if dtype == np.float32 else torch.int32
            if x.dtype == torch.float64 and tdt == torch.float32:
                warnings.warn("float64 input cast to float32 (ddks computes on float32 coordinates)", stacklevel=3)
            if x.dtype != tdt or not x.is_contiguous():
                if x.is_cuda:
                    st = _torch_stream(stream)
                    st.wait_stream(torch.cuda.current_stream(x.device))  # x is ready on the current stream
                    with torch.cuda.stream(st):
                        x = x.to(tdt).contiguous()
                    x.record_stream(st)
                else:
                    x = x.to(tdt).contiguous()
            self.keep = x
            self.ptr = x.data_ptr()
            self.shape = tuple(x.shape)
            self.is_cuda = x.is_cuda
            return
        a = np.asarray(x)
        if a.dtype == np.float64 and dtype == np.float32:
            warnings.warn("float64 input cast to float32 (ddks computes on float32 coordinates)", stacklevel=3)
        a = np.ascontiguousarray(a, dtype=dtype)
        self.keep = a
        self.ptr = a.ctypes.data
        self.shape = a.shape
        self.is_cuda = False


def _pair(P, Q, stream):
    p, q = _Arg(P, np.float32, stream), _Arg(Q, np.float32, stream)
    if len(p.shape) != 2 or len(q.shape) != 2 or p.shape[1] != q.shape[1]:
        raise ValueError(f"P {p.shape} and Q {q.shape} must be [n, d] with the same d")
    return p, q


def _batch(P, Q, stream):
    p, q = _Arg(P, np.float32, stream), _Arg(Q, np.float32, stream)
    if len(p.shape) != 3 or len(q.shape) != 3 or p.shape[0] != q.shape[0] or p.shape[2] != q.shape[2]:
        raise ValueError(f"P {p.shape} and Q {q.shape} must be [B, n, d] with the same B and d")
    return p, q


def _stream(stream):
    torch = _torch
    if stream is not None:
        if torch is not None and isinstance(stream, torch.cuda.Stream):
            return stream.cuda_stream
        return int(stream)
    if torch is not None and torch.cuda.is_available():
        return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())  # torch's current stream, raw
    return 0


# ------------------------------------------------------------------------------------------ C-ABI mirrors

def ddks_version() -> str:
    return LIB.ddks_version().decode()


def ddks_shard_range(total: int, world: int, rank: int):
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(LIB.ddks_shard_range(total, world, rank, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def ddks_get_nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(LIB.ddks_get_nccl_id(buf))
    return buf.raw


def ddks_create(device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                flags: int = DDKS_FLAG_DEFAULT) -> ctypes.c_void_p:
    ctx = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    _check(LIB.ddks_create(ctypes.byref(ctx), device, world, rank, idbuf, flags))
    return ctx


def ddks_destroy(ctx) -> None:
    _check(LIB.ddks_destroy(ctx))


def ddks_stat(ctx, P, Q, stream=None) -> Result:
    p, q = _pair(P, Q, stream)
    r = ddks_result()
    _check(LIB.ddks_stat(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1], _stream(stream), ctypes.byref(r)), ctx)
    return Result(r.num, r.den, r.D, r.argmax_origin)


_RESULT_DTYPE = np.dtype([("num", "<u8"), ("den", "<u8"), ("D", "<f8"), ("argmax_origin", "<i8")])


class BatchResult:
    """The B ddks_result structs the C call wrote, viewed as NumPy columns without per-item Python objects
    (``.num``, ``.den``, ``.D``, ``.argmax_origin``); indexing / iterating yields ``Result`` tuples."""

    def __init__(self, arr: np.ndarray):
        self.arr = arr
        self.num, self.den, self.D, self.argmax_origin = (arr[f] for f in _RESULT_DTYPE.names)

    def __len__(self):
        return len(self.arr)

    def __getitem__(self, i) -> Result:
        r = self.arr[i]
        return Result(int(r["num"]), int(r["den"]), float(r["D"]), int(r["argmax_origin"]))

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def __eq__(self, other):
        return isinstance(other, BatchResult) and self.arr.tobytes() == other.arr.tobytes()


def ddks_stat_batch(ctx, P, Q, stream=None) -> BatchResult:
    p, q = _batch(P, Q, stream)
    B = p.shape[0]
    arr = np.zeros(B, dtype=_RESULT_DTYPE)
    assert _RESULT_DTYPE.itemsize == ctypes.sizeof(ddks_result)
    _check(LIB.ddks_stat_batch(ctx, p.ptr, q.ptr, B, p.shape[1], q.shape[1], p.shape[2], _stream(stream),
                               arr.ctypes.data_as(ctypes.POINTER(ddks_result))), ctx)
    return BatchResult(arr)


def ddks_permutation_null(ctx, pooled, n_P: int, perms, stream=None):
    """-> (null_num: np.uint64 [n_perm], observed: Result, p_value: float)."""
    a = _Arg(pooled, np.float32, stream)
    pr = _Arg(perms, np.int32, stream)
    if len(a.shape) != 2:
        raise ValueError(f"pooled {a.shape} must be [n_P + n_Q, d]")
    N, d = a.shape
    n_perm = pr.shape[0] if len(pr.shape) == 2 else 0
    if n_perm and pr.shape[1] != N:
        raise ValueError(f"perms {pr.shape} must be [n_perm, {N}]")
    null = np.zeros(n_perm, dtype=np.uint64)
    obs = ddks_result()
    pv = ctypes.c_double()
    _check(LIB.ddks_permutation_null(ctx, a.ptr, n_P, N - n_P, d, pr.ptr if n_perm else None, n_perm, _stream(stream),
                                     null.ctypes.data if n_perm else None, ctypes.byref(obs), ctypes.byref(pv)), ctx)
    return null, Result(obs.num, obs.den, obs.D, obs.argmax_origin), pv.value


def ddks_stat_shard(ctx, P, Q, world: int, rank: int, stream=None) -> Result:
    """ddks_stat restricted to the origin shard rank `rank` of `world` would own (no collective)."""
    p, q = _pair(P, Q, stream)
    r = ddks_result()
    _check(LIB.ddks_stat_shard(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1], world, rank, _stream(stream),
                               ctypes.byref(r)), ctx)
    return Result(r.num, r.den, r.D, r.argmax_origin)


def ddks_stat_per_origin(ctx, P, Q, o_begin: int, o_end: int, stream=None) -> np.ndarray:
    p, q = _pair(P, Q, stream)
    out = np.zeros(max(o_end - o_begin, 0), dtype=np.uint64)
    _check(LIB.ddks_stat_per_origin(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1], o_begin, o_end,
                                    out.ctypes.data if out.size else ctypes.c_void_p(8), _stream(stream)), ctx)
    return out


def ddks_significance(ctx, P, Q, poisson: bool = False, detail: bool = False, stream=None) -> Significance:
    """Analytic significance (§3). detail=True also returns mt_hist [n_Q+1] and log_p_table [n_Q+1]."""
    p, q = _pair(P, Q, stream)
    r = ddks_significance_result()
    hist = np.zeros(q.shape[0] + 1, dtype=np.uint64) if detail else None
    table = np.zeros(q.shape[0] + 1, dtype=np.float64) if detail else None
    _check(LIB.ddks_significance(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1],
                                 DDKS_SIG_POISSON if poisson else 0, _stream(stream), ctypes.byref(r),
                                 hist.ctypes.data if detail else None, table.ctypes.data if detail else None), ctx)
    st = r.stat
    return Significance(Result(st.num, st.den, st.D, st.argmax_origin), r.S, r.log_prod, r.cells, hist, table)


def ddks_significance_batch(ctx, P, Q, poisson: bool = False, stream=None) -> list[Significance]:
    """B independent pairs P [B, n_P, d], Q [B, n_Q, d] -> one Significance per pair (no histogram/table)."""
    p, q = _batch(P, Q, stream)
    B = p.shape[0]
    out = (ddks_significance_result * B)()
    _check(LIB.ddks_significance_batch(ctx, p.ptr, q.ptr, B, p.shape[1], q.shape[1], p.shape[2],
                                       DDKS_SIG_POISSON if poisson else 0, _stream(stream), out), ctx)
    return [Significance(Result(o.stat.num, o.stat.den, o.stat.D, o.stat.argmax_origin), o.S, o.log_prod, o.cells,
                         None, None) for o in out]


def ddks_vdks(ctx, P, Q, k: int, stream=None) -> Result:
    """vdKS (Alg. 1) with k voxels per dimension."""
    p, q = _pair(P, Q, stream)
    r = ddks_result()
    _check(LIB.ddks_vdks(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1], k, _stream(stream), ctypes.byref(r)),
           ctx)
    return Result(r.num, r.den, r.D, r.argmax_origin)


def ddks_rdks(ctx, P, Q, stream=None) -> Result:
    """rdKS (Alg. 2); argmax_origin is the first corner attaining num (0 = origin, m + 1 = e_m)."""
    p, q = _pair(P, Q, stream)
    r = ddks_result()
    _check(LIB.ddks_rdks(ctx, p.ptr, p.shape[0], q.ptr, q.shape[0], p.shape[1], _stream(stream), ctypes.byref(r)), ctx)
    return Result(r.num, r.den, r.D, r.argmax_origin)


def ddks_combine_records(records) -> tuple[int, int, int]:
    """Host combine of per-rank records [(num, argmax_origin, flags), ...] -> (num, argmax_origin, flags)."""
    n = len(records)
    arr = (ddks_rank_record * n)(*[ddks_rank_record(int(a), int(b), int(c), 0) for a, b, c in records])
    out = ddks_rank_record()
    _check(LIB.ddks_combine_records(arr, n, ctypes.byref(out)))
    return int(out.num), int(out.argmax_origin), int(out.flags)


def ddks_unpad_items(gathered, total: int, world: int, n_arr: int = 1):
    """Host unpad of an all-gathered per-item block (include/ddks.h) -> (uint64 [n_arr, total], flags)."""
    g = np.ascontiguousarray(np.asarray(gathered, dtype=np.uint64))
    out = np.zeros((n_arr, total), dtype=np.uint64)
    fl = ctypes.c_uint32()
    _check(LIB.ddks_unpad_items(g.ctypes.data, total, world, n_arr, out.ctypes.data, ctypes.byref(fl)))
    return out, int(fl.value)


def gather_stride(total: int, world: int, n_arr: int = 1) -> int:
    """uint64 words per rank record of ddks_unpad_items' layout: n_arr * ceil(total / world) + 1."""
    return n_arr * (-(-total // world)) + 1


def ddks_profile_work(ctx) -> int:
    """FP32 compares the classify kernels executed since the last read (context needs DDKS_FLAG_PROFILE)."""
    v = ctypes.c_uint64()
    _check(LIB.ddks_profile_work(ctx, ctypes.byref(v)), ctx)
    return int(v.value)


def ddks_launch_count(ctx) -> int:
    return int(LIB.ddks_launch_count(ctx))


def ddks_profile_clock(ctx) -> float:
    """Mean SM MHz of the count kernels' CTAs since the last read (in-kernel clock64 / globaltimer probe)."""
    v = ctypes.c_double()
    _check(LIB.ddks_profile_clock(ctx, ctypes.byref(v)), ctx)
    return float(v.value)


def ddks_kd_levels(ctx) -> int:
    """Levels of the kd ordering used by the last count (0: position order)."""
    return int(LIB.ddks_kd_levels(ctx))


def ddks_rank_lanes(ctx) -> int:
    """1 if the last count was the rank-lane count (DESIGN.md §7 "rank lanes"), else 0."""
    return int(LIB.ddks_rank_lanes(ctx))


def ddks_profile_read(ctx):
    """-> (count_kernel_ms, count_launches, pairs) since the last read (context needs DDKS_FLAG_PROFILE)."""
    ms, n, pairs = ctypes.c_double(), ctypes.c_int64(), ctypes.c_uint64()
    _check(LIB.ddks_profile_read(ctx, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(pairs)), ctx)
    return ms.value, n.value, pairs.value


class Context:
    """RAII wrapper: ``with Context() as c: c.stat(P, Q)``."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 flags: int = DDKS_FLAG_DEFAULT):
        self.ctx = ddks_create(device, world, rank, nccl_id, flags)

    def stat(self, P, Q, stream=None) -> Result:
        return ddks_stat(self.ctx, P, Q, stream)

    def stat_batch(self, P, Q, stream=None) -> BatchResult:
        return ddks_stat_batch(self.ctx, P, Q, stream)

    def permutation_null(self, pooled, n_P, perms, stream=None):
        return ddks_permutation_null(self.ctx, pooled, n_P, perms, stream)

    def stat_shard(self, P, Q, world, rank, stream=None) -> Result:
        return ddks_stat_shard(self.ctx, P, Q, world, rank, stream)

    def stat_per_origin(self, P, Q, o_begin, o_end, stream=None):
        return ddks_stat_per_origin(self.ctx, P, Q, o_begin, o_end, stream)

    def significance(self, P, Q, poisson=False, detail=False, stream=None) -> Significance:
        return ddks_significance(self.ctx, P, Q, poisson, detail, stream)

    def significance_batch(self, P, Q, poisson=False, stream=None) -> list[Significance]:
        return ddks_significance_batch(self.ctx, P, Q, poisson, stream)

    def vdks(self, P, Q, k: int, stream=None) -> Result:
        return ddks_vdks(self.ctx, P, Q, k, stream)

    def rdks(self, P, Q, stream=None) -> Result:
        return ddks_rdks(self.ctx, P, Q, stream)

    def profile_read(self):
        return ddks_profile_read(self.ctx)

    @property
    def launch_count(self) -> int:
        return ddks_launch_count(self.ctx)

    def profile_clock(self) -> float:
        return ddks_profile_clock(self.ctx)

    def profile_work(self) -> int:
        return ddks_profile_work(self.ctx)

    @property
    def kd_levels(self) -> int:
        return ddks_kd_levels(self.ctx)

    @property
    def rank_lanes(self) -> int:
        return ddks_rank_lanes(self.ctx)

    def close(self):
        if self.ctx is not None:
            ddks_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
