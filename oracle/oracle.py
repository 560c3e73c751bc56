"""TEST INFRASTRUCTURE ONLY — the ddKS oracle (arxiv 2106.13706).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may import
this module. The product package (paper_2106_13706_b200/) never imports it, and it imports nothing from
the product: the two share no code. Inputs come from the caller as arrays.

Two independent implementations live here:

* ``ddks`` / ``per_origin`` / ``batch`` / ``permutation_null`` / ``membership`` / ``orthant_index``:
  ctypes calls into ``ddks_oracle.c`` — the paper's loop method written out in plain C,
  compares after widening float32 -> float64 (exact), int64 counts, one double division at the end.
* ``brute_force``: a definition-level pure-NumPy/Fraction implementation that never forms an orthant
  *code*: for every origin and every orthant q it evaluates the orthant predicate
  AND_k ([x_k >= o_k] == bit_k(q)) on every point (Eq. 1, Eq. 2), and compares the
  normalised counts as exact Fractions. O(2^d N^2 d): tiny inputs only.

Also the analytic significance of §3 (``log_pmf``, ``p_le``, ``significance``), written literally:
every cell's full double sum over the Delta-set band, the product as a sum of logs.

And the two approximations of §2.2.2-2.2.3 (``vdks``, Alg. 1; ``rdks``, Alg. 2), each step in the paper's order.

Plus ``ks_1d``: the classical two-sample KS statistic by a sort-merge sweep over the pooled values with
exact integers (the d=1 closed form) — used to pin the oracle, not by the oracle.

Parity-pin status: every function here is pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from itertools import product

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ddks_oracle.c")
_BUILD = os.path.join(_HERE, "build")
_SO = os.path.join(_BUILD, "libddks_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile ddks_oracle.c with gcc (-O2, OpenMP, no fast-math). Returns the .so path."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall", "-Wextra",
                               "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        c_i64, c_int, c_p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.oracle_orthant_index.argtypes = [c_p, c_p, c_int, c_int]
        lib.oracle_orthant_index.restype = c_int
        lib.oracle_membership.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_int, c_p]
        lib.oracle_membership.restype = None
        lib.oracle_ddks_per_origin.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_int, c_i64, c_i64, c_p, c_int]
        lib.oracle_ddks_per_origin.restype = c_int
        lib.oracle_ddks.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_int, c_int, c_p, c_p, c_p, c_p]
        lib.oracle_ddks.restype = c_int
        lib.oracle_ddks_batch.argtypes = [c_p, c_p, c_i64, c_i64, c_i64, c_int, c_int, c_int, c_p]
        lib.oracle_ddks_batch.restype = c_int
        lib.oracle_permutation_null.argtypes = [c_p, c_i64, c_i64, c_int, c_p, c_i64, c_int, c_int, c_p, c_p, c_p, c_p]
        lib.oracle_permutation_null.restype = c_int
        lib.oracle_log_pmf.argtypes = [c_i64, c_i64, ctypes.c_double, c_int]
        lib.oracle_log_pmf.restype = ctypes.c_double
        lib.oracle_p_le.argtypes = [ctypes.c_uint64, c_i64, c_i64, ctypes.c_double, c_int]
        lib.oracle_p_le.restype = ctypes.c_double
        lib.oracle_significance.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_int, c_int, c_int, c_p, c_p, c_p]
        lib.oracle_significance.restype = c_int
        lib.oracle_normalize_pair.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_p]
        lib.oracle_normalize_pair.restype = None
        lib.oracle_voxel_index.argtypes = [c_p, c_int, c_i64]
        lib.oracle_voxel_index.restype = c_i64
        lib.oracle_vdks.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_i64, c_p, c_p, c_p]
        lib.oracle_vdks.restype = c_int
        lib.oracle_merged_max_diff.argtypes = [c_p, c_i64, c_p, c_i64]
        lib.oracle_merged_max_diff.restype = ctypes.c_uint64
        lib.oracle_vdks_voxels.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_i64, c_i64, c_i64, c_p, c_p, c_p]
        lib.oracle_vdks_voxels.restype = c_int
        lib.oracle_rdks_corners.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_i64, c_i64, c_p, c_p, c_p, c_p]
        lib.oracle_rdks_corners.restype = c_int
        lib.oracle_rdks.argtypes = [c_p, c_i64, c_p, c_i64, c_int, c_p, c_p, c_p, c_p]
        lib.oracle_rdks.restype = c_int
        _lib = lib
    return _lib


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def orthant_index(test_point, point, ties_gt: bool = False) -> int:
    """sum_k [point_k >= test_k] 2^k (Eq. 3 '>=')."""
    t, p = _f32(test_point).ravel(), _f32(point).ravel()
    return int(_load().oracle_orthant_index(_ptr(t), _ptr(p), t.size, int(ties_gt)))


def membership(counted, test_points, ties_gt: bool = False) -> np.ndarray:
    """counts[i, q] = #{points of `counted` in orthant q about test point i}."""
    c, t = _f32(counted), _f32(test_points)
    d = c.shape[1]
    out = np.zeros((t.shape[0], 1 << d), dtype=np.int64)
    _load().oracle_membership(_ptr(c), c.shape[0], _ptr(t), t.shape[0], d, int(ties_gt), _ptr(out))
    return out


def ddks(P, Q, ties_gt: bool = False, threads: int = 0):
    """Exact ddKS -> (num, den, D, argmax_origin). D = num/den as one double division."""
    P, Q = _f32(P), _f32(Q)
    d = P.shape[1]
    num, den = ctypes.c_uint64(), ctypes.c_uint64()
    D, arg = ctypes.c_double(), ctypes.c_int64()
    rc = _load().oracle_ddks(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], d, int(ties_gt), threads,
                             ctypes.byref(num), ctypes.byref(den), ctypes.byref(D), ctypes.byref(arg))
    if rc:
        raise ValueError(f"oracle_ddks rc={rc}")
    return int(num.value), int(den.value), float(D.value), int(arg.value)


def per_origin(P, Q, o_begin: int = 0, o_end: int | None = None, ties_gt: bool = False, threads: int = 0):
    """num(o) for pooled origins [o_begin, o_end) as uint64 array."""
    P, Q = _f32(P), _f32(Q)
    N = P.shape[0] + Q.shape[0]
    o_end = N if o_end is None else o_end
    out = np.zeros(o_end - o_begin, dtype=np.uint64)
    rc = _load().oracle_ddks_per_origin(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], P.shape[1], int(ties_gt),
                                        o_begin, o_end, _ptr(out), threads)
    if rc:
        raise ValueError(f"oracle_ddks_per_origin rc={rc}")
    return out


def batch(P, Q, ties_gt: bool = False, threads: int = 0) -> np.ndarray:
    """P [B, n_P, d], Q [B, n_Q, d] -> num per item (uint64 [B]); den = n_P*n_Q for every item."""
    P, Q = _f32(P), _f32(Q)
    B, n_P, d = P.shape
    out = np.zeros(B, dtype=np.uint64)
    rc = _load().oracle_ddks_batch(_ptr(P), _ptr(Q), B, n_P, Q.shape[1], d, int(ties_gt), threads, _ptr(out))
    if rc:
        raise ValueError(f"oracle_ddks_batch rc={rc}")
    return out


def permutation_null(pooled, n_P: int, perms, ties_gt: bool = False, threads: int = 0):
    """P:L371 permutation null -> (null_num uint64 [n_perm], observed_num, p_num, p_value).
    p = p_num / (1 + n_perm), p_num = 1 + #{null_num >= observed} (add-one)."""
    pooled = _f32(pooled)
    perms = np.ascontiguousarray(np.asarray(perms, dtype=np.int32))
    N, d = pooled.shape
    n_perm = perms.shape[0]
    null = np.zeros(n_perm, dtype=np.uint64)
    obs, p_num, p_val = ctypes.c_uint64(), ctypes.c_int64(), ctypes.c_double()
    rc = _load().oracle_permutation_null(_ptr(pooled), n_P, N - n_P, d, _ptr(perms), n_perm, int(ties_gt), threads,
                                         _ptr(null), ctypes.byref(obs), ctypes.byref(p_num), ctypes.byref(p_val))
    if rc:
        raise ValueError(f"oracle_permutation_null rc={rc}")
    return null, int(obs.value), int(p_num.value), float(p_val.value)


def log_pmf(n: int, m: int, lam: float, poisson: bool = False) -> float:
    """P:L244-250 binomial pmf (or P:L278-281 Poisson pmf) of n successes in m trials at rate lam, as a log."""
    return float(_load().oracle_log_pmf(n, m, lam, int(poisson)))


def p_le(num: int, N_P: int, N_T: int, lam: float, poisson: bool = False) -> float:
    """p(d <= D) with D = num / (N_P N_T), the double sum over the Delta-set band."""
    return float(_load().oracle_p_le(num, N_P, N_T, lam, int(poisson)))


def significance(P, Q, ties_gt: bool = False, poisson: bool = False, threads: int = 0):
    """S = 1 - prod over the 2^d x N cells of p(d <= D) with lambda = (M_T + 1)/(N_T + 2).
    -> (S, log_prod, num)."""
    P, Q = _f32(P), _f32(Q)
    S, lp, num = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    rc = _load().oracle_significance(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], P.shape[1], int(ties_gt), int(poisson),
                                     threads, ctypes.byref(S), ctypes.byref(lp), ctypes.byref(num))
    if rc:
        raise ValueError(f"oracle_significance rc={rc}")
    return float(S.value), float(lp.value), int(num.value)


def normalize_pair(P, Q) -> np.ndarray:
    """Alg. 1/2 NormalizeData: pooled per-dimension (x - min)/(max - min) in double -> [N, d]."""
    P, Q = _f32(P), _f32(Q)
    out = np.zeros((P.shape[0] + Q.shape[0], P.shape[1]), dtype=np.float64)
    _load().oracle_normalize_pair(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], P.shape[1], _ptr(out))
    return out


def voxel_index(xn, k: int) -> int:
    """Alg. 1 IndexFromPoint on a normalised point: sum_m min(floor(x'_m k), k-1) k^m."""
    x = np.ascontiguousarray(np.asarray(xn, dtype=np.float64).ravel())
    return int(_load().oracle_voxel_index(_ptr(x), x.size, k))


def vdks(P, Q, k: int, v_begin: int = 0, v_end: int = -1):
    """vdKS, Alg. 1 -> (num, den, D) with D = num / den exactly as in ddks().
    [v_begin, v_end): restrict the max to filled voxels of that flat-index range (multi-rank tests)."""
    P, Q = _f32(P), _f32(Q)
    num, den, D = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
    rc = _load().oracle_vdks_voxels(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], P.shape[1], k, v_begin, v_end,
                                    ctypes.byref(num), ctypes.byref(den), ctypes.byref(D))
    if rc:
        raise ValueError(f"oracle_vdks rc={rc}")
    return int(num.value), int(den.value), float(D.value)


def merged_max_diff(c1, c2) -> int:
    """Alg. 2 GetDFromCornerLists on two ascending lists -> integer numerator over len(c1) len(c2)."""
    a = np.ascontiguousarray(np.asarray(c1, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(c2, dtype=np.float64))
    return int(_load().oracle_merged_max_diff(_ptr(a), a.size, _ptr(b), b.size))


def rdks(P, Q, c_begin: int = 0, c_end: int | None = None):
    """rdKS, Alg. 2 -> (num, den, D, arg_corner); [c_begin, c_end): corner subset (multi-rank tests)."""
    P, Q = _f32(P), _f32(Q)
    c_end = P.shape[1] + 1 if c_end is None else c_end
    num, den, D, arg = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double(), ctypes.c_int64()
    rc = _load().oracle_rdks_corners(_ptr(P), P.shape[0], _ptr(Q), Q.shape[0], P.shape[1], c_begin, c_end,
                                     ctypes.byref(num), ctypes.byref(den), ctypes.byref(D), ctypes.byref(arg))
    if rc:
        raise ValueError(f"oracle_rdks rc={rc}")
    return int(num.value), int(den.value), float(D.value), int(arg.value)


# ---------------------------------------------------------------------------------------------------
# Definition-level brute force (independent of ddks_oracle.c; tiny inputs only)
# ---------------------------------------------------------------------------------------------------

def brute_force(P, Q, ties_gt: bool = False) -> Fraction:
    """D = max over pooled origins o and orthants q of |#P_q/n_P - #Q_q/n_Q|,
    where x is in orthant q about o iff for every k: (x_k >= o_k) == bit k of q. Exact Fraction."""
    P = np.asarray(P, dtype=np.float32).astype(np.float64)
    Q = np.asarray(Q, dtype=np.float32).astype(np.float64)
    n_P, d = P.shape
    n_Q = Q.shape[0]
    origins = np.concatenate([P, Q], axis=0)
    best = Fraction(0)
    for o in origins:
        for bits in product((0, 1), repeat=d):  # bits[k] = required value of [x_k >= o_k]
            def inside(x):
                for k in range(d):
                    ge = (x[k] > o[k]) if ties_gt else (x[k] >= o[k])
                    if bool(ge) != bool(bits[k]):
                        return False
                return True
            cp = sum(1 for x in P if inside(x))
            cq = sum(1 for x in Q if inside(x))
            diff = abs(Fraction(cp, n_P) - Fraction(cq, n_Q))
            if diff > best:
                best = diff
    return best


def ks_1d(u_P, u_Q):
    """Classical two-sample KS statistic sup_t |F_P(t) - F_Q(t)| (right-continuous ECDFs) by a sort-merge
    sweep over the pooled distinct values, exact integers: returns (num, den) with D = num/den,
    num = max |cnt_P(<=t)*n_Q - cnt_Q(<=t)*n_P|, den = n_P*n_Q. Independent of the oracle."""
    a = np.sort(np.asarray(u_P, dtype=np.float32).astype(np.float64))
    b = np.sort(np.asarray(u_Q, dtype=np.float32).astype(np.float64))
    n_P, n_Q = len(a), len(b)
    i = j = 0
    best = 0
    while i < n_P or j < n_Q:
        t = min(a[i] if i < n_P else np.inf, b[j] if j < n_Q else np.inf)
        while i < n_P and a[i] == t:
            i += 1
        while j < n_Q and b[j] == t:
            j += 1
        best = max(best, abs(i * n_Q - j * n_P))
    return best, n_P * n_Q
