"""GPU parity of the two approximations of §2.2.2-2.2.3 against the oracle: vdKS (Alg. 1, voxels) and rdKS
(Alg. 2, radial corners). Both reduce to exact integers (num over den = n_P n_Q) once the f64 voxel / distance
decisions are taken in the same precision on both sides (R15-R17), so the bar is bit-exact."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


VDKS_CASES = [(300, 200, 1, 17), (1000, 900, 2, 40), (2500, 2100, 3, 12), (777, 1234, 3, 1), (1500, 1500, 4, 7),
              (900, 1100, 5, 5), (600, 500, 6, 3), (400, 450, 7, 3), (300, 320, 8, 2), (513, 257, 3, 64)]


@pytest.mark.parametrize("n_P,n_Q,d,k", VDKS_CASES)
@pytest.mark.parametrize("kind", ["normal", "mixed", "dup"])
def test_vdks_parity(ctx, n_P, n_Q, d, k, kind):
    P, Q = I.random_pair(4000 + n_P + d * 10 + k, n_P, n_Q, d, kind)
    want = O.vdks(P, Q, k)
    got = ctx.vdks(dev(P), dev(Q), k)
    assert (got.num, got.den) == want[:2] and got.D == want[2], (got, want)


# slab scans (L = k^J <= 4096 voxels per slab scanned in SMEM, then the outer dimensions in SMEM column chunks or, past
# 512 slabs, line passes; k > 4096 line passes only) and the filled-voxel list: non-power-of-two k, every J
SLAB_CASES = [(3000, 2500, 4, 17), (2000, 2200, 3, 50), (2500, 2000, 5, 10), (1500, 1800, 6, 7), (1200, 1000, 8, 4),
              (1000, 1100, 2, 300), (1500, 1200, 3, 64), (600, 700, 7, 5), (300, 250, 2, 1024), (500, 400, 1, 5000),
              (60, 50, 2, 4200), (700, 650, 3, 33)]


@pytest.mark.parametrize("n_P,n_Q,d,k", SLAB_CASES)
@pytest.mark.parametrize("kind", ["normal", "dup"])
def test_vdks_slab_parity(ctx, n_P, n_Q, d, k, kind):
    P, Q = I.random_pair(4100 + n_P + d * 10 + k, n_P, n_Q, d, kind)
    want = O.vdks(P, Q, k)
    got = ctx.vdks(dev(P), dev(Q), k)
    assert (got.num, got.den) == want[:2] and got.D == want[2], (got, want)


def test_vdks_count_buffer_reuse():
    # the slab scans leave the voxel counts zeroed for the next call, which then skips the memset over the known-zero
    # prefix: a line-pass call (k > 4096) dirties a large buffer, a small slab call cleans only its own prefix, and a
    # larger slab call must not read the rest as clean
    P2, Q2 = I.random_pair(71, 60, 50, 2, "dup")
    P3, Q3 = I.random_pair(72, 700, 650, 3, "dup")
    P4, Q4 = I.random_pair(73, 300, 250, 2, "dup")
    want = [O.vdks(P2, Q2, 4200)[:2], O.vdks(P3, Q3, 33)[:2], O.vdks(P4, Q4, 1024)[:2]]
    with K.Context() as c:
        for _ in range(2):
            assert c.vdks(dev(P2), dev(Q2), 4200)[:2] == want[0]
            assert c.vdks(dev(P3), dev(Q3), 33)[:2] == want[1]
            assert c.vdks(dev(P4), dev(Q4), 1024)[:2] == want[2]
            assert c.vdks(dev(P4), dev(Q4), 1024)[:2] == want[2]


@pytest.mark.parametrize("d,k", [(3, 64), (5, 16), (4, 23), (2, 1000), (8, 5)])
def test_vdks_aligned_vs_unaligned(ctx, d, k):
    # larger inputs than the oracle's literal SumOrthants takes in seconds: the vectorised histogram (16-byte aligned
    # inputs) and the scalar one (rows offset by one, unaligned) must agree exactly; a skewed mixture like C5's
    rng = np.random.default_rng(d * 1000 + k)
    P = rng.standard_normal((60001, d)).astype(np.float32)
    A = rng.standard_normal((50003, d))
    Q = np.where((rng.random(50003) < 0.2)[:, None], 0.3 * A + 1.0, A).astype(np.float32)
    a = ctx.vdks(dev(P), dev(Q), k)
    bufP = torch.empty(P.size + 1, dtype=torch.float32, device="cuda")
    bufQ = torch.empty(Q.size + 1, dtype=torch.float32, device="cuda")
    bufP[1:] = dev(P.ravel())
    bufQ[1:] = dev(Q.ravel())
    b = ctx.vdks(bufP[1:].view(P.shape), bufQ[1:].view(Q.shape), k)
    assert a == b and a.num > 0


def test_vdks_grid_and_edges(ctx):
    # integer grids: every point on a voxel boundary; k = #values makes vdKS the exact ddKS (oracle pin)
    rng = np.random.default_rng(8)
    for d, k in [(2, 4), (3, 5), (4, 3)]:
        P = rng.integers(0, k, (700, d)).astype(np.float32)
        Q = rng.integers(0, k, (650, d)).astype(np.float32)
        P[0], Q[0] = 0, k - 1
        got = ctx.vdks(dev(P), dev(Q), k)
        assert (got.num, got.den) == O.ddks(P, Q)[:2] == O.vdks(P, Q, k)[:2]
    # constant dimension, single points, identical samples, host inputs
    P, Q = I.random_pair(9, 50, 40, 3, "normal")
    P[:, 1] = Q[:, 1] = 2.5
    assert ctx.vdks(P, Q, 6)[:2] == O.vdks(P, Q, 6)[:2]
    assert ctx.vdks(P[:1], Q[:1], 4)[:2] == O.vdks(P[:1], Q[:1], 4)[:2]
    assert ctx.vdks(P, P.copy(), 9).num == 0
    with pytest.raises(K.DDKSError) as e:
        ctx.vdks(P, Q, 0)
    assert e.value.status == 1
    with pytest.raises(K.DDKSError) as e:
        ctx.vdks(np.zeros((3, 8), np.float32), np.ones((3, 8), np.float32), 20)
    assert e.value.status == 5


def test_vdks_c2_full(ctx):
    P, Q = I.config("C2")
    for k in (16, 32):
        got = ctx.vdks(dev(P), dev(Q), k)
        assert (got.num, got.den) == O.vdks(P, Q, k)[:2]


def test_vdks_c5_k16_vs_stored_oracle(ctx):
    # the bench's vdKS configuration (C5, k = 16) against the oracle's full literal run (Alg. 1 SumOrthants over
    # every voxel for every filled voxel; tests/golden/make_c5_vdks_oracle.py, minutes of CPU, so stored): bit-exact
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_vdks16_oracle.json")
    g = json.load(open(path))
    P, Q = I.config("C5")
    assert I.sha256_pq(P, Q) == g["input_sha256"] and g["k"] == 16
    got = ctx.vdks(dev(P), dev(Q), 16)
    assert (got.num, got.den) == (g["num"], g["den"]) and float.hex(got.D) == g["D_hex"]


def test_vdks_c5_properties(ctx):
    # full C5 (10^6 + 10^6, d = 5, k = 16): the oracle's literal SumOrthants is O(F k^d); use properties that hold
    # at any size: symmetry and power-of-two scale invariance (NormalizeData removes it exactly)
    P, Q = I.config("C5")
    a = ctx.vdks(dev(P), dev(Q), 16)
    assert a == ctx.vdks(dev(Q), dev(P), 16)
    s = np.array([2, 4, 0.5, 1, 8], np.float32)
    assert a == ctx.vdks(dev(P * s), dev(Q * s), 16)
    assert 0 < a.num <= a.den


# ------------------------------------------------------------------------------------------------ rdKS (Alg. 2)

RDKS_CASES = [(300, 200, 1), (1000, 900, 2), (5000, 4000, 3), (777, 1234, 4), (2100, 2500, 5), (600, 500, 8),
              (100, 100, 64), (100, 100, 1000), (4096, 1, 3), (1, 4097, 2)]


@pytest.mark.parametrize("n_P,n_Q,d", RDKS_CASES)
@pytest.mark.parametrize("kind", ["normal", "mixed", "dup"])
def test_rdks_parity(ctx, n_P, n_Q, d, kind):
    P, Q = I.random_pair(7000 + n_P + d, n_P, n_Q, d, kind)
    want = O.rdks(P, Q)
    got = ctx.rdks(dev(P), dev(Q))
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3]) and got.D == want[2], (got, want)


def test_rdks_ties_and_edges(ctx):
    rng = np.random.default_rng(12)
    # integer grids: many exactly equal distances (tie groups spanning radix tiles)
    for d, k, n in [(2, 3, 9000), (3, 2, 6000), (5, 3, 3000)]:
        P = rng.integers(0, k, (n, d)).astype(np.float32)
        Q = rng.integers(0, k, (n - 7, d)).astype(np.float32)
        want = O.rdks(P, Q)
        got = ctx.rdks(dev(P), dev(Q))
        assert (got.num, got.argmax_origin) == (want[0], want[3])
    P, Q = I.random_pair(13, 60, 50, 3, "normal")
    P[:, 2] = Q[:, 2] = -1.25  # constant dimension -> 0.5
    assert ctx.rdks(P, Q)[:2] == O.rdks(P, Q)[:2]
    assert ctx.rdks(P, P.copy()).num == 0
    assert ctx.rdks(P, Q).num == ctx.rdks(Q, P).num
    Pn = P.copy()
    Pn[3, 1] = np.inf
    with pytest.raises(K.DDKSError) as e:
        ctx.rdks(Pn, Q)
    assert e.value.status == 4


def test_rdks_count_buffer_reuse():
    # the sweep re-zeroes every bucket count it reads (k_rdb_cand / k_rdb_finish), so a completed call leaves the
    # count buffer clean and the next call skips its memset over the known-zero prefix; a larger call must still
    # zero the rest, and a call that falls back to the full sort (flag 256) must leave the buffer marked dirty
    rng = np.random.default_rng(7)
    Pf = np.concatenate([rng.random((200, 2)), 0.5 + 1e-4 * rng.random((10000, 2))]).astype(np.float32)
    Qf = np.concatenate([rng.random((300, 2)), 0.5 + 1e-4 * rng.random((9000, 2)) + 2e-5]).astype(np.float32)
    Pf[0], Qf[0] = 0.0, 1.0
    cases = [I.random_pair(81, 3000, 2000, 3, "normal"), I.random_pair(82, 40000, 30000, 2, "mixed"),
             (Pf, Qf), I.random_pair(83, 9000, 11000, 4, "dup"), I.random_pair(84, 500, 700, 5, "grid")]
    want = [O.rdks(P, Q) for P, Q in cases]
    with K.Context() as c:
        for _ in range(2):
            for (P, Q), w in zip(cases, want):
                got = c.rdks(dev(P), dev(Q))
                assert (got.num, got.den, got.argmax_origin) == (w[0], w[1], w[3]), (got, w)


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_rdks_configs_full(ctx, name):
    # full-size parity: the oracle's rdKS is O((d+1) N log N) too, so it runs on whole BASELINE configs
    P, Q = I.config(name)
    want = O.rdks(P, Q)
    got = ctx.rdks(dev(P), dev(Q))
    assert (got.num, got.den, got.argmax_origin) == (want[0], want[1], want[3])


def test_rdks_pruned_equals_full_sort_and_fallback(ctx):
    # the bucket-pruned sweep (default) against the full radix sort path, and a workload whose maximum sits in a
    # bucket with more than 4096 keys and several distinct distances (forces the in-call fallback to the full sort)
    with K.Context(flags=K.DDKS_FLAG_RDKS_FULL_SORT) as cf:
        for seed, (n_P, n_Q, d, kind) in enumerate([(3000, 2000, 3, "normal"), (700, 900, 2, "grid"),
                                                    (5000, 5000, 5, "mixed"), (100, 100, 300, "dup")]):
            P, Q = I.random_pair(7700 + seed, n_P, n_Q, d, kind)
            assert ctx.rdks(dev(P), dev(Q)) == cf.rdks(dev(P), dev(Q))
        rng = np.random.default_rng(7)
        P = np.concatenate([rng.random((200, 2)), 0.5 + 1e-4 * rng.random((10000, 2))]).astype(np.float32)
        Q = np.concatenate([rng.random((300, 2)), 0.5 + 1e-4 * rng.random((9000, 2)) + 2e-5]).astype(np.float32)
        P[0], Q[0] = 0.0, 1.0
        want = O.rdks(P, Q)
        got = ctx.rdks(dev(P), dev(Q))
        assert (got.num, got.argmax_origin) == (want[0], want[3]) and got == cf.rdks(dev(P), dev(Q))


def test_vdks_validates_in_place(ctx):
    # vdKS reads the caller's arrays in place (no pack): the min/max pass rejects NaN / Inf and treats -0 as +0
    P, Q = I.random_pair(61, 500, 400, 3, "normal")
    for bad in (np.nan, np.inf, -np.inf):
        Pb = P.copy()
        Pb[123, 1] = bad
        with pytest.raises(K.DDKSError) as e:
            ctx.vdks(dev(Pb), dev(Q), 8)
        assert e.value.status == 4
    Pz, Qz = P.copy(), Q.copy()
    Pz[:50, 0] = -0.0
    Qz[:50, 0] = 0.0
    for k in (4, 7, 16):
        assert ctx.vdks(dev(Pz), dev(Qz), k)[:2] == O.vdks(Pz, Qz, k)[:2]
        assert ctx.vdks(Pz, Qz, k)[:2] == O.vdks(Pz, Qz, k)[:2]  # host inputs
