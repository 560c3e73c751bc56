"""GPU parity of the round-2 execution paths (through the C-ABI, against the oracle):

* the accumulate mode's partials: zeroed once at allocation, and k_finalize re-zeroes what it reads (no memset per
  call) -- across many consecutive segmented calls of changing shape on one context;
* the fused packed-key argmax ((num / g) << 31 | (2^31 - 1 - origin), R7) against the per-origin +
  k_argmax path (DDKS_NO_KEY, test only) on position-ordered, kd-ordered, sharded and significance counts;
* origin blocks chunked over several launches on grid.y (DDKS_GRIDY lowers the 65535 chunk, test only);
* K = 4 kd levels forced through the context flag alone (DDKS_FLAG_KD_LEVELS is 3 bits wide);
* the in-kernel executed-compare counter (ddks_profile_work) the bench's executed_frac is built from.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def want_of(P, Q, ties_gt=False):
    w = O.ddks(P, Q, ties_gt=ties_gt)
    return (w[0], w[1], w[3])


def test_partials_left_clean_across_calls():
    # segmented counts (several point segments per origin block) of changing shapes on ONE context: every call must
    # find the int32 partials zero, i.e. every k_finalize cleared what the previous call accumulated
    cases = [(9000, 7000, 3, "normal"), (3000, 5000, 8, "grid"), (9000, 7000, 3, "mixed"), (12000, 12000, 5, "dup"),
             (700, 900, 2, "grid"), (9000, 7000, 3, "normal"), (4000, 4100, 6, "mixed")]
    with K.Context(flags=K.DDKS_FLAG_NO_X0) as c:
        for i, (n_P, n_Q, d, kind) in enumerate(cases):
            P, Q = I.random_pair(31000 + i, n_P, n_Q, d, kind)
            got = c.stat(dev(P), dev(Q))
            assert (got.num, got.den, got.argmax_origin) == want_of(P, Q), (i, got)
            # batch items and the significance's SPLIT count share the same partial buffers
            if i % 3 == 0:
                Pb, Qb = P[: 3 * 500].reshape(3, 500, d), Q[: 3 * 400].reshape(3, 400, d)
                assert [r.num for r in c.stat_batch(dev(Pb), dev(Qb))] == O.batch(Pb, Qb).tolist()


@pytest.mark.parametrize("flags,n_P,n_Q,d,kind", [
    (K.DDKS_FLAG_NO_X0, 3000, 2500, 3, "grid"), (K.DDKS_FLAG_NO_X0, 9000, 7001, 5, "mixed"),
    (K.DDKS_FLAG_FORCE_X0, 9000, 7001, 5, "grid"), (K.DDKS_FLAG_FORCE_X0, 4000, 3000, 8, "dup"),
    (K.DDKS_FLAG_NO_X0 | K.DDKS_FLAG_FORCE_DIRECT, 1500, 1300, 4, "normal"), (K.DDKS_FLAG_NO_X0, 5, 300, 2, "grid")])
def test_packed_key_argmax_equals_k_argmax_path(monkeypatch, flags, n_P, n_Q, d, kind):
    P, Q = I.random_pair(32000 + n_P + d, n_P, n_Q, d, kind)
    want = want_of(P, Q)
    with K.Context(flags=flags) as c:
        a = c.stat(dev(P), dev(Q))
        monkeypatch.setenv("DDKS_NO_KEY", "1")
        b = c.stat(dev(P), dev(Q))
        parts = [c.stat_shard(dev(P), dev(Q), 3, r) for r in range(3)]
        sb = c.significance(dev(P[:600]), dev(Q[:500]))
        monkeypatch.delenv("DDKS_NO_KEY")
        parts_k = [c.stat_shard(dev(P), dev(Q), 3, r) for r in range(3)]
        sa = c.significance(dev(P[:600]), dev(Q[:500]))
    assert (a.num, a.den, a.argmax_origin) == want == (b.num, b.den, b.argmax_origin)
    assert parts == parts_k
    comb = K.ddks_combine_records([(p.num, p.argmax_origin, 0) for p in parts])
    assert comb == (want[0], want[2], 0)
    assert sa.stat == sb.stat and (sa.stat.num, sa.stat.argmax_origin) == (lambda w: (w[0], w[3]))(O.ddks(P[:600], Q[:500]))
    assert sa.log_prod == sb.log_prod


def test_argmax_beyond_the_key_range():
    # n_P n_Q / gcd >= 2^33: the packed key cannot hold num / g, the library takes the per-origin + k_argmax path
    n_P, n_Q = 100_003, 100_019  # coprime: g = 1, n_P n_Q ~ 1.0e10 > 2^33
    rng = np.random.default_rng(33)
    P = rng.integers(0, 50, (n_P, 2)).astype(np.float32)
    Q = rng.integers(0, 50, (n_Q, 2)).astype(np.float32)
    with K.Context() as c:
        got = c.stat(dev(P), dev(Q))
    # argmax: num attained there (oracle on that one origin) and by no smaller sampled origin
    assert got.den == n_P * n_Q and 0 < got.num <= got.den
    assert int(O.per_origin(P, Q, got.argmax_origin, got.argmax_origin + 1)[0]) == got.num
    per = O.per_origin(P, Q, 0, min(got.argmax_origin, 4000))
    assert (per < got.num).all()


@pytest.mark.parametrize("flags", [K.DDKS_FLAG_NO_X0, K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(3),
                                   K.DDKS_FLAG_NO_X0 | K.DDKS_FLAG_FORCE_DIRECT])
def test_origin_blocks_chunked_on_grid_y(monkeypatch, flags):
    P, Q = I.random_pair(33100, 14000, 11000, 4, "mixed")
    want = want_of(P, Q)
    monkeypatch.setenv("DDKS_GRIDY", "3")
    with K.Context(flags=flags) as c:
        got = c.stat(dev(P), dev(Q))
        for w in (2, 3):
            parts = [c.stat_shard(dev(P), dev(Q), w, r) for r in range(w)]
            assert K.ddks_combine_records([(p.num, p.argmax_origin, 0) for p in parts])[:2] == (want[0], want[2])
        sig = c.significance(dev(P[:3000]), dev(Q[:2000]))
    assert (got.num, got.den, got.argmax_origin) == want
    assert sig.stat.num == O.ddks(P[:3000], Q[:2000])[0]


def test_kd_four_levels_from_the_flag_alone(monkeypatch):
    monkeypatch.delenv("DDKS_KD", raising=False)
    P, Q = I.random_pair(33200, 30000, 26000, 5, "normal")
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(4)) as c:
        got = c.stat(dev(P), dev(Q))
        assert c.kd_levels == 4
    assert (got.num, got.den, got.argmax_origin) == want_of(P, Q)


def test_executed_compares_counter():
    P, Q = I.random_pair(33300, 20000, 20000, 5, "normal")
    N, d = 40000, 5
    with K.Context(flags=K.DDKS_FLAG_PROFILE | K.DDKS_FLAG_NO_X0 | K.DDKS_FLAG_NO_RANK) as c:  # the FP32 count
        c.stat(dev(P), dev(Q))
        ms, n, pairs = c.profile_read()
        ex = c.profile_work()
        assert pairs == N * N
        # position order: every lane compares all d dims against every point; the clamped tail slots of the last
        # origin block (a whole number of warps' origins past N) compare too
        assert ex % (d * N) == 0
        slots = ex // (d * N)
        assert N <= slots < N + 4096 and slots % 256 == 0, slots
        assert c.profile_work() == 0  # reset by the read
    with K.Context(flags=K.DDKS_FLAG_PROFILE | K.DDKS_FLAG_FORCE_X0) as c:
        c.stat(dev(P), dev(Q))
        ms, n, pairs = c.profile_read()
        ex = c.profile_work()
        assert c.kd_levels >= 2
        assert (d - c.kd_levels) * pairs < ex < d * pairs  # decided bits are not compares; the undecided dims are
    with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
        Pb, Qb = I.random_pair(33301, 64 * 512, 64 * 512, 4, "normal")
        c.stat_batch(dev(Pb.reshape(64, 512, 4)), dev(Qb.reshape(64, 512, 4)))
        ms, n, pairs = c.profile_read()
        ex = c.profile_work()
        assert 3 * pairs < ex < 4 * pairs  # warp-level bit 0 decisions


SMALL_CASES = [(1, 1, 1, "normal"), (200, 200, 3, "normal"), (37, 41, 2, "grid"), (300, 5, 5, "mixed"),
               (4096, 4096, 3, "grid"), (4000, 4192, 8, "mixed"), (2, 8190, 4, "dup"), (129, 127, 6, "grid"),
               (3000, 1000, 7, "normal"), (1023, 1025, 1, "grid")]


@pytest.mark.parametrize("n_P,n_Q,d,kind", SMALL_CASES)
def test_small_fused_path(monkeypatch, n_P, n_Q, d, kind):
    # the one-launch small-N statistic (raw input, cluster of point segments, DSMEM counter reduction, per-block
    # records reduced on the host) against the oracle and against the packed multi-launch path
    P, Q = I.random_pair(34000 + n_P + d, n_P, n_Q, d, kind)
    want = want_of(P, Q)
    with K.Context() as c:
        for _ in range(3):  # uncaptured, captured, replayed
            got = c.stat(dev(P), dev(Q))
            assert (got.num, got.den, got.argmax_origin) == want, got
        assert c.stat(P, Q) == got  # host inputs (H2D inside the call)
        monkeypatch.setenv("DDKS_NO_SMALL", "1")
        assert c.stat(dev(P), dev(Q)) == got
        monkeypatch.delenv("DDKS_NO_SMALL")
    with K.Context(flags=K.DDKS_FLAG_TIES_GT) as c:
        got = c.stat(dev(P), dev(Q))
        assert (got.num, got.den, got.argmax_origin) == want_of(P, Q, ties_gt=True)


def test_small_fused_path_nonfinite_and_window():
    P, Q = I.random_pair(34100, 500, 600, 3, "normal")
    with K.Context() as c:
        for bad in (np.nan, np.inf, -np.inf):
            Qb = Q.copy()
            Qb[599, 2] = bad  # the last row of the last segment
            with pytest.raises(K.DDKSError) as e:
                c.stat(dev(P), dev(Qb))
            assert e.value.status == 4
        assert (lambda r: (r.num, r.den, r.argmax_origin))(c.stat(dev(P), dev(Q))) == want_of(P, Q)
    # n_P, n_Q coprime and unbalanced: N * max(a, b) > 32767, so the fused path is skipped (counter window)
    P, Q = I.random_pair(34101, 97, 1201, 2, "grid")
    with K.Context() as c:
        r = c.stat(dev(P), dev(Q))
    assert (r.num, r.den, r.argmax_origin) == want_of(P, Q)


MMA_CASES = [(512, 512, 4, 1000, "normal"), (37, 41, 1, 300, "grid"), (200, 150, 2, 257, "mixed"),
             (500, 333, 3, 256, "grid"), (130, 190, 5, 40, "dup"), (100, 123, 6, 511, "normal"),
             (70, 60, 7, 9, "grid"), (1, 1, 3, 5, "normal"), (1500, 1200, 4, 64, "mixed"), (3, 61, 2, 700, "grid")]


@pytest.mark.parametrize("n_P,n_Q,d,n_perm,kind", MMA_CASES)
def test_tensor_core_null(monkeypatch, n_P, n_Q, d, n_perm, kind):
    # the label-invariant null as a tcgen05 contraction (one-hot orthant matrix x label matrix, fp16 -> fp32 TMEM)
    # against the oracle and against the SMEM-counter kernel (DDKS_NO_MMA); ragged N (not a multiple of 64), ragged
    # n_perm (not a multiple of 256), empty origin rows of the last tile, ties
    P, Q = I.random_pair(35000 + n_P + d, n_P, n_Q, d, kind)
    pooled = np.concatenate([P, Q])
    N = n_P + n_Q
    rng = np.random.default_rng(35000 + n_perm)
    perms = np.stack([rng.permutation(N) for _ in range(n_perm)]).astype(np.int32)
    o_null, o_obs, _, o_p = O.permutation_null(pooled, n_P, perms)
    with K.Context() as c:
        null, obs, p = c.permutation_null(dev(pooled), n_P, dev(perms))
        monkeypatch.setenv("DDKS_NO_MMA", "1")
        null2, obs2, p2 = c.permutation_null(dev(pooled), n_P, dev(perms))
        monkeypatch.delenv("DDKS_NO_MMA")
    assert np.array_equal(null, o_null) and obs.num == o_obs and p == o_p
    assert np.array_equal(null2, o_null) and p2 == p
    with K.Context(flags=K.DDKS_FLAG_TIES_GT) as c:
        null_gt, _, _ = c.permutation_null(dev(pooled), n_P, dev(perms))
    assert np.array_equal(null_gt, O.permutation_null(pooled, n_P, perms, ties_gt=True)[0])


def test_tensor_core_null_rejects_bad_rows():
    P, Q = I.random_pair(35100, 100, 90, 3, "normal")
    pooled = np.concatenate([P, Q])
    perms = np.stack([np.random.default_rng(i).permutation(190) for i in range(20)]).astype(np.int32)
    perms[7, 3] = perms[7, 4]  # a duplicate index: not a permutation
    with K.Context() as c:
        with pytest.raises(K.DDKSError) as e:
            c.permutation_null(dev(pooled), 100, dev(perms))
        assert e.value.status == 1



@pytest.mark.parametrize("mma", [True, False])
def test_permutation_groups(monkeypatch, mma):
    # permutations processed in groups (bounded label-image / bitmap memory): group boundaries inside tensor-core
    # tiles and label words, the last group ragged; identical to one group and to the oracle
    P, Q = I.random_pair(37000, 300, 250, 4, "grid")
    pooled = np.concatenate([P, Q])
    rng = np.random.default_rng(37001)
    perms = np.stack([rng.permutation(550) for _ in range(601)]).astype(np.int32)
    if not mma:
        monkeypatch.setenv("DDKS_NO_MMA", "1")
    o_null, o_obs, _, o_p = O.permutation_null(pooled, 300, perms)
    with K.Context() as c:
        one = c.permutation_null(dev(pooled), 300, dev(perms))
        monkeypatch.setenv("DDKS_PERM_GROUP", "257")
        grp = c.permutation_null(dev(pooled), 300, dev(perms))
    assert np.array_equal(one[0], o_null) and np.array_equal(grp[0], o_null)
    assert one[1].num == grp[1].num == o_obs and one[2] == grp[2] == o_p
