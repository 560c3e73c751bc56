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


def test_rank_lane_shards():
    P, Q = I.random_pair(32100, 7000, 6000, 8, "grid")
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
    # the captured call graph replays the rank-lane count (and reports it); SPLIT-only sizes and the > convention
    # take the FP32 counts
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
    with K.Context(flags=RANK) as c:
        r = c.stat(dev(P1), dev(Q1))
        assert c.rank_lanes == 0 and (r.num, r.argmax_origin) == (O.ddks(P1, Q1)[0], O.ddks(P1, Q1)[3])


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
