"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element on the same seeded inputs.
The bar is bit-exact: num and den are integers, D is the same single IEEE division, argmax is the smallest
pooled index attaining num (R7). Every test here needs a B200 (``-m gpu``)."""
import json
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


@pytest.fixture(scope="module")
def ctx():
    c = K.Context()
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_direct():
    c = K.Context(flags=K.DDKS_FLAG_FORCE_DIRECT)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_gt():
    c = K.Context(flags=K.DDKS_FLAG_TIES_GT)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_pair(ctx, P, Q, ties_gt=False, host=False):
    want = O.ddks(P, Q, ties_gt=ties_gt)
    got = ctx.stat(P if host else dev(P), Q if host else dev(Q))
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3]), (got, want)
    assert got.D == want[2] and np.float64(got.D).tobytes() == np.float64(want[2]).tobytes()
    return got


# ----------------------------------------------------------------------------------- worked examples

def test_spec_and_hand_examples(ctx, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["statistic"]:
        P, Q = np.array(c["P"], np.float32), np.array(c["Q"], np.float32)
        r = ctx.stat(dev(P), dev(Q))
        assert r.num * c["D_den"] == r.den * c["D_num"], c["cite"]
    h = json.load(open(os.path.join(golden_dir, "hand_examples.json")))
    for c in h["cases"]:
        P, Q = np.array(c["P"], np.float32), np.array(c["Q"], np.float32)
        check_pair(ctx, P, Q)
        r = ctx.stat(dev(P), dev(Q))
        assert (r.num, r.den) == (c["ge"]["num"], c["ge"]["den"]), c["name"]


def test_tie_flag(ctx_gt):
    h = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))
    for c in h["cases"]:
        if "gt" in c:
            r = ctx_gt.stat(dev(np.array(c["P"], np.float32)), dev(np.array(c["Q"], np.float32)))
            assert (r.num, r.den) == (c["gt"]["num"], c["gt"]["den"])


# ----------------------------------------------------------------------------------- random parity

SIZES = [(1, 1), (1, 7), (2, 3), (31, 33), (200, 200), (255, 257), (511, 513), (997, 1009), (1000, 2000),
         (1500, 700), (2047, 2049)]


@pytest.mark.parametrize("d", range(1, 9))
@pytest.mark.parametrize("kind", ["normal", "grid", "mixed", "dup"])
def test_random_parity_all_d(ctx, ctx_direct, d, kind):
    for i, (n_P, n_Q) in enumerate(SIZES):
        if d >= 7 and n_P * n_Q > 1_200_000:
            continue
        P, Q = I.random_pair(1000 * d + 17 * i + 13 * ["normal", "grid", "mixed", "dup"].index(kind), n_P, n_Q, d, kind)
        check_pair(ctx, P, Q)
        if i % 3 == 0:
            check_pair(ctx_direct, P, Q)


@pytest.mark.parametrize("d", [1, 3, 5, 8])
def test_random_parity_ties_gt(ctx_gt, d):
    for i, (n_P, n_Q) in enumerate([(33, 31), (500, 700), (1200, 1200)]):
        P, Q = I.random_pair(77 + i + d, n_P, n_Q, d, "grid")
        check_pair(ctx_gt, P, Q, ties_gt=True)


def test_host_pointer_path_equals_device(ctx):
    P, Q = I.random_pair(5, 3000, 2500, 5, "mixed")
    a = check_pair(ctx, P, Q, host=True)
    b = ctx.stat(dev(P), dev(Q))
    assert a == b
    c = ctx.stat(torch.from_numpy(P), torch.from_numpy(Q))  # CPU tensors -> host path
    assert c == b


def test_per_origin_export(ctx):
    for d in (2, 5, 8):
        P, Q = I.random_pair(40 + d, 1300, 1100, d, "mixed")
        N = 2400
        want = O.per_origin(P, Q)
        got = ctx.stat_per_origin(dev(P), dev(Q), 0, N)
        assert np.array_equal(got, want)
        got = ctx.stat_per_origin(P, Q, 1299, 1302)
        assert np.array_equal(got, want[1299:1302])


def test_symmetry_identity_on_gpu(ctx):
    for d in (1, 4, 6):
        P, Q = I.random_pair(90 + d, 800, 600, d, "normal")
        a, b = ctx.stat(dev(P), dev(Q)), ctx.stat(dev(Q), dev(P))
        assert (a.num, a.den, a.D) == (b.num, b.den, b.D)
        assert ctx.stat(dev(P), dev(P)).num == 0


def test_split_counter_mode_sampled():
    # n_P*n_Q/gcd >= 2^31 forces separate c_P, c_Q counters (SPLIT mode); check sampled origins one by one.
    n_P, n_Q = 50_000, 49_999
    P, Q = I.random_pair(3, n_P, n_Q, 3, "mixed")
    with K.Context() as c:
        idx = [0, 1, 2, 49_999, 50_000, 50_001, 99_998]
        for o in idx:
            assert int(c.stat_per_origin(dev(P), dev(Q), o, o + 1)[0]) == int(O.per_origin(P, Q, o, o + 1)[0]), o
        r = c.stat(dev(P), dev(Q))
        assert r.den == n_P * n_Q and 0 < r.num <= r.den
        r2 = c.stat(dev(Q), dev(P))
        assert r2.num == r.num


# ----------------------------------------------------------------------------------- errors / edge cases

def test_errors(ctx):
    P = np.zeros((4, 3), np.float32)
    bad = P.copy()
    bad[2, 1] = np.nan
    with pytest.raises(K.DDKSError) as e:
        ctx.stat(dev(bad), dev(P))
    assert e.value.status == 4
    bad[2, 1] = np.inf
    with pytest.raises(K.DDKSError) as e:
        ctx.stat(dev(P), dev(bad))
    assert e.value.status == 4
    with pytest.raises(K.DDKSError) as e:
        ctx.stat(dev(P), dev(np.zeros((0, 3), np.float32)))
    assert e.value.status == 2
    with pytest.raises(K.DDKSError) as e:
        ctx.stat(dev(np.zeros((4, 9), np.float32)), dev(np.zeros((4, 9), np.float32)))
    assert e.value.status == 3
    # context still usable after errors
    check_pair(ctx, *I.random_pair(1, 10, 12, 3, "grid"))
    # invalid permutation rows
    pooled = np.random.default_rng(0).standard_normal((10, 2)).astype(np.float32)
    perms = np.stack([np.arange(10), np.arange(10)]).astype(np.int32)
    perms[1, 3] = 4  # duplicate
    with pytest.raises(K.DDKSError) as e:
        ctx.permutation_null(dev(pooled), 5, dev(perms))
    assert e.value.status == 1
    perms[1, 3] = 10  # out of range
    with pytest.raises(K.DDKSError):
        ctx.permutation_null(dev(pooled), 5, dev(perms))


def test_extreme_values(ctx):
    f = np.float32
    cases = [
        (np.array([[-0.0]], f), np.array([[0.0]], f)),
        (np.array([[1.401298464324817e-45]], f), np.array([[2.802596928649634e-45]], f)),
        (np.array([[3.4e38, -3.4e38], [1.0, 1.0]], f), np.array([[-3.4e38, 3.4e38], [np.nextafter(f(1), f(2)), 1.0]], f)),
        (np.full((600, 4), 7.0, f), np.full((300, 4), 7.0, f)),  # all identical -> D = 0
    ]
    for P, Q in cases:
        check_pair(ctx, P, Q)


# ----------------------------------------------------------------------------------- batch / permutation

def test_batch_parity(ctx, ctx_direct):
    rng = np.random.default_rng(21)
    for (B, n_P, n_Q, d) in [(1, 5, 6, 2), (7, 33, 31, 4), (40, 128, 128, 3), (5, 700, 300, 5), (3, 90, 100, 8)]:
        P = rng.standard_normal((B, n_P, d)).astype(np.float32)
        Q = (rng.standard_normal((B, n_Q, d)) * 1.2).astype(np.float32)
        Q[:, ::3] = np.round(Q[:, ::3])
        want = O.batch(P, Q)
        for c in (ctx, ctx_direct):
            got = c.stat_batch(dev(P), dev(Q))
            assert [r.num for r in got] == want.tolist()
            assert all(r.den == n_P * n_Q for r in got)


@pytest.fixture(scope="module")
def ctx_gather():
    c = K.Context(flags=K.DDKS_FLAG_PERM_GATHER)
    yield c
    c.close()


@pytest.mark.parametrize("d", range(1, 9))
def test_permutation_parity(ctx, ctx_gather, d):
    # default path: label-invariant (one classification per pair for J permutations); gather path: relabel + recount
    rng = np.random.default_rng(22 + d)
    for (n_P, n_Q, n_perm) in [(20, 21, 33), (100, 80, 50), (301, 299, 17), (1, 6, 5)]:
        pooled = rng.standard_normal((n_P + n_Q, d)).astype(np.float32)
        pooled[::4] = np.round(pooled[::4])
        perms = np.stack([np.arange(n_P + n_Q)] + [rng.permutation(n_P + n_Q) for _ in range(n_perm - 1)]).astype(np.int32)
        null, obs, p_num, p = O.permutation_null(pooled, n_P, perms)
        for c in (ctx, ctx_gather):
            g_null, g_obs, g_p = c.permutation_null(dev(pooled), n_P, dev(perms))
            assert np.array_equal(g_null, null) and g_obs.num == obs and g_p == p, (d, n_P, n_Q)
    g_null2, _, _ = ctx.permutation_null(pooled, n_P, perms)  # host inputs
    assert np.array_equal(g_null2, null)


def test_permutation_ties_gt(ctx_gt):
    rng = np.random.default_rng(5)
    pooled = rng.integers(0, 3, (60, 3)).astype(np.float32)
    perms = np.stack([rng.permutation(60) for _ in range(40)]).astype(np.int32)
    null, obs, _, p = O.permutation_null(pooled, 25, perms, ties_gt=True)
    g_null, g_obs, g_p = ctx_gt.permutation_null(dev(pooled), 25, dev(perms))
    assert np.array_equal(g_null, null) and g_obs.num == obs and g_p == p


# ----------------------------------------------------------------------------------- BASELINE configs

def test_config_c1_c2_c3_full(ctx):
    for name in ("C1", "C2", "C3"):
        P, Q = I.config(name)
        check_pair(ctx, P, Q)


def test_config_c4_every_item_and_permutation(ctx, golden_dir):
    # full C4 in the bench's launch configuration: EVERY one of the 4096 batch items and EVERY one of the 1000
    # null permutations element by element against the oracle's full run (tests/golden/c4_oracle.json, written by
    # make_c4_oracle.py from oracle/ only and pinned to the survey's independent aggregates in test_oracle_pins.py),
    # plus a live oracle run on a seeded sample of items and permutations
    g = json.load(open(os.path.join(golden_dir, "c4_oracle.json")))
    P, Q = I.config("C4")
    assert I.sha256_pq(P, Q) == g["input_sha256"]
    got = ctx.stat_batch(dev(P), dev(Q))
    nums = np.array([r.num for r in got], dtype=np.uint64)
    want = np.array(g["batch_num"], dtype=np.uint64)
    bad = np.nonzero(nums != want)[0]
    assert bad.size == 0, (bad[:10], nums[bad[:10]], want[bad[:10]])
    assert all(r.den == g["den"] and r.D == r.num / g["den"] for r in got)
    rng = np.random.default_rng(44)
    idx = np.sort(rng.choice(4096, 96, replace=False))
    assert nums[idx].tolist() == O.batch(P[idx], Q[idx]).tolist()
    perms = I.c4_perms()
    pooled = np.concatenate([P[I.C4_PERM_PAIR], Q[I.C4_PERM_PAIR]])
    null, obs, p = ctx.permutation_null(dev(pooled), 512, dev(perms))
    want_null = np.array(g["null_num"], dtype=np.uint64)
    bad = np.nonzero(null != want_null)[0]
    assert bad.size == 0, (bad[:10], null[bad[:10]], want_null[bad[:10]])
    assert obs.num == g["observed_num"] and p == g["p_value"]
    jdx = np.sort(rng.choice(1000, 48, replace=False))
    o_null, o_obs, _, _ = O.permutation_null(pooled, 512, perms[jdx])
    assert np.array_equal(null[jdx], o_null) and o_obs == obs.num


def test_config_c5_sampled(ctx):
    # full size, the bench's launch configuration; sampled origins checked one by one against the oracle
    P, Q = I.config("C5")
    dP, dQ = dev(P), dev(Q)
    rng = np.random.default_rng(5)
    idx = sorted(set([0, 1, 2, 3, 999_999, 1_000_000, 1_000_001, 1_999_999, 123_456, 1_765_432]
                     + rng.integers(0, 2_000_000, 22).tolist()))
    for o in idx:
        got = int(ctx.stat_per_origin(dP, dQ, o, o + 1)[0])
        assert got == int(O.per_origin(P, Q, o, o + 1)[0]), o
    r = ctx.stat(dP, dQ)
    assert r.den == 10**12 and 0 < r.num <= r.den
    # the reported max is attained at the reported argmax origin (checked by the oracle) ...
    assert int(O.per_origin(P, Q, r.argmax_origin, r.argmax_origin + 1)[0]) == r.num
    # ... and no sampled origin exceeds it
    assert all(int(O.per_origin(P, Q, o, o + 1)[0]) <= r.num for o in idx[:8])
    # the bench's x0-ordered kernel and the position-ordered kernel agree on the whole statistic (num and argmax)
    with K.Context(flags=K.DDKS_FLAG_NO_X0) as c:
        assert c.stat(dP, dQ) == r


# ----------------------------------------------------------------------------------- x0-ordered count (bit-0 elision)

@pytest.fixture(scope="module")
def ctx_nox0():
    c = K.Context(flags=K.DDKS_FLAG_NO_X0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_x0():
    c = K.Context(flags=K.DDKS_FLAG_FORCE_X0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_x0_gt():
    c = K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_TIES_GT)
    yield c
    c.close()


X0_CASES = [(300, 200, 2, "grid"), (1500, 1300, 3, "normal"), (5000, 4000, 2, "grid"), (6000, 6000, 3, "mixed"), (4500, 5200, 4, "normal"), (9000, 7001, 5, "grid"),
            (5000, 5000, 5, "dup"), (4096, 4096, 6, "mixed"), (20000, 1, 3, "normal"), (3, 12000, 5, "grid"),
            (3000, 2500, 7, "mixed"), (2600, 3100, 8, "normal"), (1500, 1500, 8, "grid"), (40000, 30000, 2, "normal")]


@pytest.mark.parametrize("n_P,n_Q,d,kind", X0_CASES)
def test_x0_ordered_parity(ctx_x0, ctx_nox0, n_P, n_Q, d, kind):
    # FORCE_X0 and 2 <= d <= 6 takes the x0-ordered kernel (tiles whose x_0 range does not interleave with the
    # CTA's origins skip the dim-0 compare); tie-heavy grids put many equal x_0 values on CTA and tile boundaries
    P, Q = I.random_pair(9100 + n_P + d, n_P, n_Q, d, kind)
    if kind == "grid":
        P[:, 0] = np.round(P[:, 0] * 3) / 3
    got = check_pair(ctx_x0, P, Q)
    assert ctx_nox0.stat(dev(P), dev(Q)) == got


@pytest.mark.parametrize("d", [2, 5])
def test_x0_ordered_ties_gt(ctx_x0_gt, d):
    P, Q = I.random_pair(9300 + d, 6000, 5000, d, "grid")
    want = O.ddks(P, Q, ties_gt=True)
    got = ctx_x0_gt.stat(dev(P), dev(Q))
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3])


# ----------------------------------------------------------------------------------- kd-ordered count (K levels)

KD_CASES = [(2, "2,5,1", 9000, 7000, 2, "normal"), (2, "2,3,1", 6000, 6000, 3, "grid"), (3, "3,3,2", 12000, 9000, 3, "mixed"),
            (3, "3,2,2", 8000, 8000, 4, "grid"), (3, "3,3,3", 16000, 14000, 5, "mixed"), (2, "2,7,1", 20000, 17001, 5, "dup"),
            (3, "3,2,3", 9000, 9000, 6, "normal"), (3, "3,3,3", 7000, 6000, 7, "grid"), (2, "2,4,1", 5000, 5400, 8, "mixed"),
            (3, "3,9,9", 4000, 3000, 5, "normal"), (3, "3,3,3", 3, 12000, 5, "grid"), (2, "2,2,1", 20000, 1, 3, "normal"),
            (2, "2,1,1", 9000, 7000, 2, "grid"), (3, None, 11000, 9000, 5, "mixed"),
            (4, "4,2,2,2", 12000, 9000, 5, "mixed"), (4, "4,3,2,2", 9000, 8000, 4, "grid"),
            (4, "4,2,3,2", 8000, 7000, 8, "normal"), (4, "4,5,5,5", 4000, 3000, 6, "normal"),
            (4, "4,2,2,3", 3, 9000, 7, "grid")]


@pytest.mark.parametrize("K_,env,n_P,n_Q,d,kind", KD_CASES)
def test_kd_ordered_parity(monkeypatch, ctx_nox0, K_, env, n_P, n_Q, d, kind):
    # K levels of kd ordering (bits 0..K-1 decided per tile where the tile's box does not interleave with the CTA's
    # origins'); DDKS_KD fixes the level and the slab / cell counts so small inputs still get several cells (and
    # empty ones: 3,9,9 and 4,5,5,5)
    if env is None:
        monkeypatch.delenv("DDKS_KD", raising=False)
    else:
        monkeypatch.setenv("DDKS_KD", env)
    P, Q = I.random_pair(9500 + n_P + 3 * d, n_P, n_Q, d, kind)
    if kind == "grid":
        P[:, :3] = np.round(P[:, :3] * 3) / 3
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(K_)) as c:
        got = check_pair(c, P, Q)
        assert c.kd_levels == K_
    assert ctx_nox0.stat(dev(P), dev(Q)) == got


def test_kd_ties_gt_uses_one_level(monkeypatch):
    # the '>' test convention is instantiated with one level: a forced K falls back to 1, still exact
    monkeypatch.setenv("DDKS_KD", "3,3,3")
    P, Q = I.random_pair(9400, 7000, 6000, 5, "grid")
    want = O.ddks(P, Q, ties_gt=True)
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_TIES_GT | K.DDKS_FLAG_KD_LEVELS(3)) as c:
        got = c.stat(dev(P), dev(Q))
        assert c.kd_levels == 1
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3])


@pytest.mark.parametrize("K_,env", [(2, "2,4,1"), (3, "3,3,2"), (4, "4,2,2,2")])
def test_kd_shard_rehearsal(monkeypatch, K_, env):
    # origin shards are positions of the kd order: max over shards and the smallest attaining argmax reproduce the
    # oracle for any world size
    monkeypatch.setenv("DDKS_KD", env)
    P, Q = I.random_pair(9950 + K_, 15000, 13000, 5, "mixed")
    want = O.ddks(P, Q)
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(K_)) as c:
        for world in (2, 3, 8):
            parts = [c.stat_shard(dev(P), dev(Q), world, r) for r in range(world)]
            num = max(p.num for p in parts)
            arg = min(p.argmax_origin for p in parts if p.num == num)
            assert (num, arg) == (want[0], want[3]), (world, parts)


# ----------------------------------------------------------------------------------- warp-level x0 batch count

@pytest.mark.parametrize("B,n_P,n_Q,d,kind", [(37, 512, 512, 4, "normal"), (9, 700, 300, 3, "grid"), (5, 1024, 1024, 5, "mixed"),
                                              (11, 33, 97, 8, "dup"), (6, 1, 200, 2, "grid"), (3, 1000, 17, 6, "normal"),
                                              (4, 129, 257, 7, "grid")])
def test_batch_warp_x0_parity(B, n_P, n_Q, d, kind):
    # ddks_stat_batch on small items sorts every label run by x_0 (k_pack_sorted) and decides bit 0 per warp and
    # 32-point sub-tile (k_count<WX>); against the oracle and the unsorted position-ordered path (DDKS_FLAG_NO_X0)
    P, Q = I.random_pair(7100 + B + d, B * n_P, B * n_Q, d, kind)
    if kind == "grid":
        P[:, 0] = np.round(P[:, 0] * 2) / 2
    P, Q = P.reshape(B, n_P, d), Q.reshape(B, n_Q, d)
    want = O.batch(P, Q).tolist()
    with K.Context() as c, K.Context(flags=K.DDKS_FLAG_NO_X0) as cn:
        got = [r.num for r in c.stat_batch(dev(P), dev(Q))]
        assert got == want
        assert [r.num for r in cn.stat_batch(dev(P), dev(Q))] == want


# ----------------------------------------------------------------------------------- launch-limit edge paths

def test_batch_beyond_grid_z_limit(ctx):
    # B > 65535 items: the library runs the items in grid.z chunks of 65535
    rng = np.random.default_rng(17)
    B = 70_001
    P = rng.integers(0, 3, (B, 4, 2)).astype(np.float32)
    Q = rng.integers(0, 3, (B, 3, 2)).astype(np.float32)
    got = ctx.stat_batch(dev(P), dev(Q))
    want = O.batch(P, Q)
    assert np.array_equal(got.num, want) and np.all(got.den == 12)


def test_permutation_null_beyond_label_path(ctx):
    # N > 65535 pooled points: the label-invariant kernel's 16-bit counters do not apply, so the library gathers
    # each relabelled sample and re-runs the full classification (x0 / position-ordered count)
    rng = np.random.default_rng(19)
    n_P, n_Q = 33_000, 33_001
    pooled = np.round(rng.standard_normal((n_P + n_Q, 1)) * 50).astype(np.float32)  # d = 1, tie-heavy
    perms = np.stack([np.arange(n_P + n_Q), rng.permutation(n_P + n_Q)]).astype(np.int32)
    null, obs, p = ctx.permutation_null(dev(pooled), n_P, dev(perms))
    o_null, o_obs, o_pnum, o_p = O.permutation_null(pooled, n_P, perms)
    assert np.array_equal(null, o_null) and obs.num == o_obs and p == o_p


def test_config_c5_full_vs_stored_oracle(ctx):
    # the whole C5 statistic against the oracle's own full run (tests/golden/make_c5_oracle.py; hours of CPU, so
    # stored): num, den, D bits and argmax, bit for bit
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_oracle.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c5_oracle.json not generated yet")
    g = json.load(open(path))
    P, Q = I.config("C5")
    assert I.sha256_pq(P, Q) == g["input_sha256"]
    r = ctx.stat(dev(P), dev(Q))
    assert (r.num, r.den, r.argmax_origin) == (g["num"], g["den"], g["argmax_origin"])
    assert float.hex(r.D) == g["D_hex"]


@pytest.mark.parametrize("flags,n_P,n_Q,d", [(0, 3000, 2500, 3), (64, 3000, 2500, 3), (64, 9000, 7000, 5),
                                               (0, 1200, 1300, 8), (64, 150, 170, 2)])
def test_shard_rehearsal_combines_to_the_statistic(flags, n_P, n_Q, d):
    # ddks_stat_shard runs the exact kernels on the origin shard a rank would own (x0 order when FORCE_X0 = 64);
    # max over shards and the smallest attaining argmax must reproduce ddks_stat and the oracle for any world size
    P, Q = I.random_pair(9900 + n_P + d, n_P, n_Q, d, "mixed")
    want = O.ddks(P, Q)
    with K.Context(flags=flags) as c:
        full = c.stat(dev(P), dev(Q))
        assert (full.num, full.argmax_origin) == (want[0], want[3])
        for world in (2, 3, 8):
            parts = [c.stat_shard(dev(P), dev(Q), world, r) for r in range(world)]
            num = max(p.num for p in parts)
            arg = min(p.argmax_origin for p in parts if p.num == num)
            assert (num, arg) == (want[0], want[3]), (world, parts)


def test_profile_clock_probe():
    # DDKS_FLAG_PROFILE: the count kernel's per-CTA clock64 / %globaltimer probe yields the SM clock it ran at
    P, Q = I.random_pair(77, 20000, 20000, 5, "normal")
    with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
        c.stat(dev(P), dev(Q))
        mhz = c.profile_clock()
        assert 300.0 < mhz < 3000.0, mhz
        assert c.profile_clock() == 0.0  # reset by the read
    with K.Context() as c:
        c.stat(dev(P), dev(Q))
        assert c.profile_clock() == 0.0  # no probe without the flag


@pytest.mark.parametrize("n_P,n_Q,d,kind", [(12000, 11000, 8, "normal"), (15000, 14000, 3, "mixed"),
                                            (21000, 19500, 5, "grid")])
def test_default_mid_n_kd_path(n_P, n_Q, d, kind):
    # sizes just above the default kd thresholds (d = 8 from 20 000 rows, d = 3 from 28 000, d = 5 from 40 000) whose
    # sample-size ratios need SPLIT counters: without the rank lanes the unforced call takes the kd count with the
    # cluster mid-N ordering; with them (the default at d = 5..8 here) the two-launch SPLIT rank-lane count. Both must
    # equal the oracle bit for bit
    P, Q = I.random_pair(9700 + d, n_P, n_Q, d, kind)
    if kind == "grid":
        P[:, :2] = np.round(P[:, :2] * 4) / 4
        Q[:, :2] = np.round(Q[:, :2] * 4) / 4
    with K.Context() as c:
        check_pair(c, P, Q)
        assert (c.rank_lanes == 1 and c.kd_levels == 0) if d >= 5 else (c.kd_levels >= 1 and c.rank_lanes == 0)
    with K.Context(flags=K.DDKS_FLAG_NO_RANK) as c:
        check_pair(c, P, Q)
        assert c.kd_levels >= 1 and c.rank_lanes == 0
