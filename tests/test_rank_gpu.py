"""GPU parity of the rank-lane count (csrc/ddks_rank.cuh; DESIGN.md §7 "rank lanes"): every (origin, point) pair is
classified from 10-bit per-CTA rank lanes instead of FP32 compares, which must give exactly the statistic of the
definition (Eq. 3, bit k = [x_k >= o_k]; Eq. 6). Compared with the CPU oracle element by
element: num, den, the D bits, the argmax origin and the per-origin nums; tie-heavy, ragged and sharded cases."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

RANK = K.DDKS_FLAG_FORCE_RANK


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(c, P, Q, want=None):
    want = want or O.ddks(P, Q)
    got = c.stat(dev(P), dev(Q))
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3]), (got, want)
    assert np.float64(got.D).tobytes() == np.float64(want[2]).tobytes()
    return got


# N > 8192 (the small geometry ends there) with DIFF counters (max(n_P, n_Q) / gcd <= 7): ragged origin blocks
# (N % 384 != 0), equal and unequal sample sizes; 7000 + 6000 (a = 6, b = 7, lcm 42 000 > 32 767) needs several
# int16 windows, so its counters are flushed in chunks of 12 tiles
SIZES = [(4100, 4100), (5001, 3334), (6144, 6144), (7000, 6000)]


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", ["normal", "grid", "mixed", "dup"])
def test_rank_lane_parity(d, kind):
    with K.Context(flags=RANK) as c, K.Context(flags=RANK | K.DDKS_FLAG_FORCE_DIRECT) as cd:
        for i, (n_P, n_Q) in enumerate(SIZES):
            P, Q = I.random_pair(31000 + 100 * d + 7 * i + 11 * ["normal", "grid", "mixed", "dup"].index(kind), n_P, n_Q, d, kind)
            want = O.ddks(P, Q)
            check(c, P, Q, want)
            assert c.rank_lanes == 1
            if i % 2 == 0:
                check(cd, P, Q, want)  # one point segment: the in-kernel finalisation


@pytest.mark.parametrize("d", [3, 5, 6, 8])
def test_rank_lane_per_origin(d):
    P, Q = I.random_pair(32000 + d, 5200, 3900, d, "mixed")
    want = O.per_origin(P, Q)
    with K.Context(flags=RANK) as c:
        got = c.stat_per_origin(dev(P), dev(Q), 0, 9100)
        assert c.rank_lanes == 1
        assert np.array_equal(got, want)
        got = c.stat_per_origin(dev(P), dev(Q), 383, 4000)  # a range that starts inside an origin block
        assert np.array_equal(got, want[383:4000])


@pytest.mark.parametrize("n_P,n_Q", [(7000, 6000), (7000, 6001)])  # DIFF counters; SPLIT counters
def test_rank_lane_shards(n_P, n_Q):
    P, Q = I.random_pair(32100, n_P, n_Q, 8, "grid")
    want = O.ddks(P, Q)
    with K.Context(flags=RANK) as c:
        check(c, P, Q, want)
        assert c.rank_lanes == 1
        for world in (2, 3, 8):
            parts = [c.stat_shard(dev(P), dev(Q), world, r) for r in range(world)]
            num = max(p.num for p in parts)
            arg = min(p.argmax_origin for p in parts if p.num == num)
            assert (num, arg) == (want[0], want[3]), (world, parts)


def test_rank_lane_extreme_values():
    # denormals, signed zeros, 1-ulp neighbours, huge magnitudes and many exact ties in one input: the per-CTA
    # ranks must order them exactly as the IEEE >= of the oracle
    rng = np.random.default_rng(32200)
    vals = np.array([0.0, -0.0, 2.0 ** -149, -(2.0 ** -149), 2.0 ** -126, 1.0, np.nextafter(np.float32(1), np.float32(2)),
                     -1.0, 3.0e38, -3.0e38, 1e-30, 7.0], np.float32)
    P = vals[rng.integers(0, len(vals), (4800, 8))].astype(np.float32)
    Q = vals[rng.integers(0, len(vals), (4000, 8))].astype(np.float32)
    Q[:, 3] = rng.standard_normal(4000).astype(np.float32)
    with K.Context(flags=RANK) as c:
        check(c, P, Q)
        assert c.rank_lanes == 1
        check(c, P[:, :3].copy(), Q[:, :3].copy())  # one rank word per point
        check(c, P[:, :5].copy(), Q[:, :5].copy())  # two
        assert c.rank_lanes == 1


def test_rank_lane_is_the_default_at_d8_and_equals_the_fp32_paths():
    # d = 8, N = 60 000: the default call takes the rank-lane count (no kd ordering); the position-ordered FP32 count
    # and the kd-ordered count give the same statistic, argmax and per-origin nums
    P, Q = I.random_pair(32300, 30000, 30000, 8, "normal")
    with K.Context() as c, K.Context(flags=K.DDKS_FLAG_NO_RANK | K.DDKS_FLAG_NO_X0) as cf, \
            K.Context(flags=K.DDKS_FLAG_NO_RANK) as ck:
        a = c.stat(dev(P), dev(Q))
        assert c.kd_levels == 0 and c.rank_lanes == 1
        b = cf.stat(dev(P), dev(Q))
        k = ck.stat(dev(P), dev(Q))
        assert ck.kd_levels >= 1 and ck.rank_lanes == 0 and cf.rank_lanes == 0
        assert a == b == k
        pa = c.stat_per_origin(dev(P), dev(Q), 20000, 21000)
        pb = cf.stat_per_origin(dev(P), dev(Q), 20000, 21000)
        assert np.array_equal(pa, pb)
        # and a sample of origins against the oracle's per-origin definition
        assert np.array_equal(pa[:64], O.per_origin(P, Q, 20000, 20064))


def test_rank_lane_default_at_d7_mid_n():
    # d = 7, N = 22 000 (below the kd threshold, inside the rank-lane range): the unforced call takes the rank lanes
    P, Q = I.random_pair(9707, 11000, 11000, 7, "mixed")
    with K.Context() as c:
        check(c, P, Q)
        assert c.kd_levels == 0 and c.rank_lanes == 1


def test_rank_lane_graph_replay_and_fallbacks():
    # the captured call graph replays the rank-lane count (and reports it); the > convention and small N take the
    # FP32 counts; sizes that need SPLIT counters take the two-launch SPLIT rank-lane count
    P, Q = I.random_pair(32400, 6000, 5000, 8, "mixed")
    want = O.ddks(P, Q)
    dP, dQ = dev(P), dev(Q)
    with K.Context() as c:
        for _ in range(4):
            r = c.stat(dP, dQ)
            assert (r.num, r.argmax_origin) == (want[0], want[3]) and c.rank_lanes == 1
    with K.Context(flags=K.DDKS_FLAG_TIES_GT) as c:
        r = c.stat(dP, dQ)
        assert c.rank_lanes == 0 and r.num == O.ddks(P, Q, ties_gt=True)[0]
    P1, Q1 = I.random_pair(32401, 9000, 7, 8, "normal")  # a = 9000 / gcd: DIFF counters would overflow -> SPLIT
    with K.Context() as c:
        for _ in range(3):
            r = c.stat(dev(P1), dev(Q1))
            assert c.rank_lanes == 1 and (r.num, r.argmax_origin) == (O.ddks(P1, Q1)[0], O.ddks(P1, Q1)[3])
    with K.Context(flags=K.DDKS_FLAG_NO_RANK) as c:
        r = c.stat(dev(P1), dev(Q1))
        assert c.rank_lanes == 0 and (r.num, r.argmax_origin) == (O.ddks(P1, Q1)[0], O.ddks(P1, Q1)[3])
    P2, Q2 = I.random_pair(32402, 3000, 2000, 8, "normal")  # N <= 8192: the fused small-N statistic
    with K.Context(flags=RANK) as c:
        r = c.stat(dev(P2), dev(Q2))
        assert c.rank_lanes == 0 and r.num == O.ddks(P2, Q2)[0]


def _fuzz_cases(seed, n):
    # DIFF-counter sizes n_P = m b', n_Q = m a' (a', b' <= 7) with 8192 < N <= ~15 000, so origin blocks, tiles and
    # the P / Q boundary fall at arbitrary offsets; lcm > 32 767 for the larger ratios (several flush windows)
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        a, b = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        m = int(rng.integers(8193 // (a + b) + 1, 15000 // (a + b) + 1))
        out.append((m * b, m * a, int(rng.integers(2, 9)), str(rng.choice(["normal", "grid", "mixed", "dup"])),
                    int(rng.integers(0, 2 ** 31))))
    return out


@pytest.mark.parametrize("n_P,n_Q,d,kind,seed", _fuzz_cases(2025, int(os.environ.get("DDKS_FUZZ_CASES", "36")) // 3))
def test_rank_lane_fuzz(n_P, n_Q, d, kind, seed):
    P, Q = I.random_pair(seed, n_P, n_Q, d, kind)
    with K.Context(flags=RANK) as c:
        check(c, P, Q)
        assert c.rank_lanes == 1


# ---------------------------------------------------------------------------------------- SPLIT counters
# sample sizes whose DIFF counters would overflow (max(n_P, n_Q) / gcd > 7) and the significance's M_T histogram: the
# rank-lane count keeps c_P and c_Q apart (P rows and Q rows in two launches, +1 per pair; Eq. 5)

SPLIT_SIZES = [(4100, 4093), (5000, 7001), (9001, 3000), (300, 8000)]


@pytest.mark.parametrize("d", [2, 3, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", ["normal", "grid", "dup"])
def test_rank_lane_split_parity(d, kind):
    with K.Context(flags=RANK) as c:
        for i, (n_P, n_Q) in enumerate(SPLIT_SIZES):
            P, Q = I.random_pair(34000 + 100 * d + 7 * i + 11 * ["normal", "grid", "dup"].index(kind), n_P, n_Q, d, kind)
            check(c, P, Q)
            assert c.rank_lanes == 1


def test_rank_lane_split_window_and_per_origin():
    # n_P = 40 000 > 32 767: the P pass flushes its 16-bit counters in two windows; per-origin nums of a range
    P, Q = I.random_pair(34500, 40000, 1201, 6, "mixed")
    want = O.per_origin(P, Q, 39000, 41201)
    with K.Context(flags=RANK) as c, K.Context(flags=K.DDKS_FLAG_NO_RANK | K.DDKS_FLAG_NO_X0) as cf:
        got = c.stat_per_origin(dev(P), dev(Q), 39000, 41201)
        assert c.rank_lanes == 1
        assert np.array_equal(got, want)
        assert c.stat(dev(P), dev(Q)) == cf.stat(dev(P), dev(Q))
        assert c.rank_lanes == 1 and cf.rank_lanes == 0


@pytest.mark.parametrize("n_P,n_Q,d,kind", [(4200, 4100, 8, "normal"), (5000, 5000, 6, "grid"), (3000, 6000, 7, "mixed"),
                                            (4500, 4000, 3, "dup")])
def test_rank_lane_significance(n_P, n_Q, d, kind):
    # the significance through the SPLIT rank-lane count: the M_T histogram equals the oracle's membership counts
    # (P:L208-209), statistic and argmax equal the oracle's, and log_prod is bit-identical to the FP32 count's
    P, Q = I.random_pair(34600 + d, n_P, n_Q, d, kind)
    with K.Context(flags=RANK) as c, K.Context(flags=K.DDKS_FLAG_NO_RANK | K.DDKS_FLAG_NO_X0) as cf:
        a = c.significance(dev(P), dev(Q), detail=True)
        assert c.rank_lanes == 1
        b = cf.significance(dev(P), dev(Q), detail=True)
        assert cf.rank_lanes == 0
    assert a.stat == b.stat and np.array_equal(a.mt_hist, b.mt_hist) and a.log_prod == b.log_prod
    pooled = np.concatenate([P, Q])
    MT = O.membership(Q, pooled)
    assert np.array_equal(a.mt_hist, np.bincount(MT.ravel(), minlength=n_Q + 1).astype(np.uint64))
    want = O.ddks(P, Q)
    assert (a.stat.num, a.stat.argmax_origin) == (want[0], want[3])
