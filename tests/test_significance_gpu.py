"""GPU parity of the analytic significance (§3) against the oracle.

Integers (num, den, argmax and the M_T histogram) must match bit for bit. The floating-point parts (the per-m
factor log p(d <= D | lambda_m), log_prod and S) carry the tolerance DESIGN.md §3 R14 derives from the arithmetic:
both sides evaluate log pmf = log m! - log n! - log (m-n)! + n log l + (m-n) log(1-l) from lgamma values of
magnitude up to L = lgamma(n_max + 1), so each pmf carries a relative error of a few ulps of L; the oracle also
rounds the literal sum p over (N_P + 1)(N_T + 1) terms before taking its log (the GPU sums the complement). Per
table entry:  tol_entry = 32 eps (1 + L) + (N_P + 1)(N_T + 1) eps,  and over the 2^d N cells: cells x tol_entry.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

EPS = np.finfo(np.float64).eps


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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def tol_entry(n_P, n_Q):
    L = math.lgamma(max(n_P, n_Q) + 1)
    return 32 * EPS * (1 + L) + (n_P + 1) * (n_Q + 1) * EPS


def oracle_hist(P, Q):
    pooled = np.concatenate([P, Q])
    MT = O.membership(Q, pooled)  # [N, 2^d] Q-counts about every pooled test point
    return np.bincount(MT.ravel(), minlength=Q.shape[0] + 1).astype(np.uint64)


CASES = [(37, 29, 1, "normal"), (40, 30, 2, "grid"), (64, 64, 3, "normal"), (50, 70, 3, "mixed"),
         (90, 60, 4, "normal"), (33, 41, 5, "dup")]


@pytest.mark.parametrize("n_P,n_Q,d,kind", CASES)
@pytest.mark.parametrize("poisson", [False, True])
def test_significance_parity_small(ctx, n_P, n_Q, d, kind, poisson):
    P, Q = I.random_pair(1000 + 7 * n_P + d, n_P, n_Q, d, kind)
    S_o, lp_o, num_o = O.significance(P, Q, poisson=poisson)
    g = ctx.significance(dev(P), dev(Q), poisson=poisson, detail=True)
    want = O.ddks(P, Q)
    assert (g.stat.num, g.stat.den, g.stat.argmax_origin) == (want[0], want[1], want[3])
    assert g.stat.num == num_o and g.cells == (1 << d) * (n_P + n_Q)
    # the M_T histogram: exact
    assert np.array_equal(g.mt_hist, oracle_hist(P, Q))
    # every tabulated factor against the oracle's literal double sum
    te = tol_entry(n_P, n_Q)
    for m in np.nonzero(g.mt_hist)[0]:
        lam = (m + 1.0) / (n_Q + 2.0)
        ref = math.log(O.p_le(num_o, n_P, n_Q, lam, poisson))
        assert abs(g.log_p_table[m] - ref) <= te, (m, g.log_p_table[m], ref)
    tol = g.cells * te
    assert abs(g.log_prod - lp_o) <= tol + 1e-12 * abs(lp_o), (g.log_prod, lp_o, tol)
    assert abs(g.S - S_o) <= tol + 1e-12, (g.S, S_o)
    assert 0.0 <= g.S <= 1.0


def test_significance_direct_equals_segmented(ctx, ctx_direct):
    # N > the int16 flush window (32767) forces the segmented accumulate path; the in-kernel direct finaliser
    # must give the same histogram and bit-identical log_prod (same table, same fixed-order reduction)
    P, Q = I.random_pair(77, 20000, 15000, 3, "mixed")
    a = ctx.significance(dev(P), dev(Q), detail=True)
    b = ctx_direct.significance(dev(P[:9000]), dev(Q[:7000]), detail=True)
    c = ctx.significance(dev(P[:9000]), dev(Q[:7000]), detail=True)
    assert np.array_equal(b.mt_hist, c.mt_hist) and b.log_prod == c.log_prod and b.stat == c.stat
    N = 35000
    assert int(a.mt_hist.sum()) == 8 * N
    # every test point's Q-counts sum to n_Q over its 2^d orthants
    assert int((np.arange(a.mt_hist.size, dtype=np.uint64) * a.mt_hist).sum()) == N * 15000
    assert np.array_equal(a.mt_hist, oracle_hist(P, Q))
    assert a.stat.num == O.ddks(P, Q)[0]


def test_significance_c2_sampled(ctx):
    # BASELINE config C2 (d=3, 10^4 + 10^4): exact histogram and num; table entries sampled against the oracle
    P, Q = I.config("C2")
    g = ctx.significance(dev(P), dev(Q), detail=True)
    want = O.ddks(P, Q)
    assert (g.stat.num, g.stat.argmax_origin) == (want[0], want[3])
    assert np.array_equal(g.mt_hist, oracle_hist(P, Q))
    nz = np.nonzero(g.mt_hist)[0]
    rng = np.random.default_rng(5)
    te = tol_entry(10_000, 10_000)
    for m in [int(nz[0]), int(rng.choice(nz))]:
        ref = math.log(O.p_le(g.stat.num, 10_000, 10_000, (m + 1.0) / 10_002.0))
        assert abs(g.log_p_table[m] - ref) <= te, (m, g.log_p_table[m], ref)
    assert 0.0 <= g.S <= 1.0 and g.log_prod <= 0.0


def test_significance_closed_forms(ctx):
    rng = np.random.default_rng(32)
    # fully separated samples: D = 1, every factor is 1 -> S = 0
    P = rng.random((12, 2)).astype(np.float32)
    Q = (rng.random((10, 2)) + 2).astype(np.float32)
    g = ctx.significance(dev(P), dev(Q))
    assert g.stat.num == 120 and g.log_prod == 0.0 and g.S == 0.0
    # identical samples: D = 0, S close to 1
    P = rng.random((50, 3)).astype(np.float32)
    g = ctx.significance(dev(P), dev(P.copy()))
    assert g.stat.num == 0 and g.S > 0.9
    # host inputs == device inputs
    P, Q = I.random_pair(9, 80, 60, 2, "normal")
    assert ctx.significance(P, Q) == ctx.significance(dev(P), dev(Q))


def test_significance_errors(ctx):
    P = np.zeros((4, 2), np.float32)
    with pytest.raises(K.DDKSError) as e:
        ctx.significance(P, np.zeros((0, 2), np.float32))
    assert e.value.status == 2
    Pn = P.copy()
    Pn[1, 1] = np.nan
    with pytest.raises(K.DDKSError) as e:
        ctx.significance(Pn, P)
    assert e.value.status == 4


@pytest.mark.parametrize("n_P,n_Q,d,kind", [(40, 30, 2, "grid"), (64, 64, 3, "normal"), (90, 60, 4, "normal"),
                                            (33, 41, 5, "dup"), (30, 26, 8, "mixed")])
def test_significance_x0_ordered(n_P, n_Q, d, kind):
    # the x0-ordered SPLIT kernel (bin-0 elision; the bench's C5 significance path) against the oracle and the
    # position-ordered kernel: identical histogram and statistic, bit-identical log_prod
    P, Q = I.random_pair(1000 + 7 * n_P + d, n_P, n_Q, d, kind)
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0) as cx, K.Context(flags=K.DDKS_FLAG_NO_X0) as cn:
        a = cx.significance(dev(P), dev(Q), detail=True)
        b = cn.significance(dev(P), dev(Q), detail=True)
    assert a.stat == b.stat and np.array_equal(a.mt_hist, b.mt_hist) and a.log_prod == b.log_prod
    assert np.array_equal(a.mt_hist, oracle_hist(P, Q))
    want = O.ddks(P, Q)
    assert (a.stat.num, a.stat.argmax_origin) == (want[0], want[3])


@pytest.mark.parametrize("K_,env,n_P,n_Q,d", [(2, "2,3,1", 3000, 2600, 3), (3, "3,3,2", 4000, 3500, 5),
                                               (3, "3,2,2", 2500, 2500, 8), (4, "4,2,2,2", 4000, 3600, 6)])
def test_significance_kd_ordered(monkeypatch, K_, env, n_P, n_Q, d):
    # the kd-ordered SPLIT kernel with several slabs / cells: identical M_T histogram, statistic and log_prod
    monkeypatch.setenv("DDKS_KD", env)
    P, Q = I.random_pair(1300 + n_P + d, n_P, n_Q, d, "mixed")
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(K_)) as cx, \
            K.Context(flags=K.DDKS_FLAG_NO_X0) as cn:
        a = cx.significance(dev(P), dev(Q), detail=True)
        assert cx.kd_levels == K_
        b = cn.significance(dev(P), dev(Q), detail=True)
    assert a.stat == b.stat and np.array_equal(a.mt_hist, b.mt_hist) and a.log_prod == b.log_prod
    want = O.ddks(P, Q)
    assert (a.stat.num, a.stat.argmax_origin) == (want[0], want[3])


def test_significance_x0_c2(ctx):
    P, Q = I.config("C2")
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0) as cx:
        a = cx.significance(dev(P), dev(Q), detail=True)
    b = ctx.significance(dev(P), dev(Q), detail=True)
    assert a.stat == b.stat and np.array_equal(a.mt_hist, b.mt_hist) and a.log_prod == b.log_prod


@pytest.mark.parametrize("n_P,n_Q,d", [(40, 30, 2), (35, 45, 4), (30, 26, 6)])
def test_significance_ties_gt(n_P, n_Q, d):
    # the '>' convention (DDKS_FLAG_TIES_GT, test only) through both the position- and the x0-ordered SPLIT kernels
    P, Q = I.random_pair(1500 + n_P + d, n_P, n_Q, d, "grid")
    S_o, lp_o, num_o = O.significance(P, Q, ties_gt=True)
    MT = O.membership(Q, np.concatenate([P, Q]), ties_gt=True)
    h_o = np.bincount(MT.ravel(), minlength=n_Q + 1).astype(np.uint64)
    for fl in (K.DDKS_FLAG_TIES_GT, K.DDKS_FLAG_TIES_GT | K.DDKS_FLAG_FORCE_X0):
        with K.Context(flags=fl) as c:
            g = c.significance(dev(P), dev(Q), detail=True)
        assert g.stat.num == num_o and np.array_equal(g.mt_hist, h_o)
        assert abs(g.log_prod - lp_o) <= g.cells * tol_entry(n_P, n_Q) + 1e-12 * abs(lp_o)


@pytest.mark.parametrize("B,n_P,n_Q,d,poisson", [(7, 40, 30, 2, False), (5, 50, 50, 3, True), (3, 33, 41, 5, False),
                                                 (4, 30, 26, 8, False)])
def test_significance_batch(ctx, B, n_P, n_Q, d, poisson):
    # B independent pairs in one call: each item against the oracle, and bit-identical to the single-pair call
    Pb, Qb = I.random_pair(2000 + B + d, B * n_P, B * n_Q, d, "mixed")
    Pb, Qb = Pb.reshape(B, n_P, d), Qb.reshape(B, n_Q, d)
    got = ctx.significance_batch(dev(Pb), dev(Qb), poisson=poisson)
    te = tol_entry(n_P, n_Q)
    for b in range(B):
        S_o, lp_o, num_o = O.significance(Pb[b], Qb[b], poisson=poisson)
        g = got[b]
        assert g.stat.num == num_o and g.stat.den == n_P * n_Q and g.cells == (1 << d) * (n_P + n_Q)
        assert abs(g.log_prod - lp_o) <= g.cells * te + 1e-12 * abs(lp_o), (b, g.log_prod, lp_o)
        one = ctx.significance(dev(Pb[b]), dev(Qb[b]), poisson=poisson)
        assert one.stat.num == g.stat.num and one.log_prod == g.log_prod and one.S == g.S


def test_significance_batch_many_small(ctx):
    # the paper's power-analysis shape: many 50 + 50 tests in 3-D; spot-check items against the oracle
    rng = np.random.default_rng(77)
    B = 512
    Pb = rng.random((B, 50, 3)).astype(np.float32)
    Qb = rng.random((B, 50, 3)).astype(np.float32)
    Qb[B // 2:] = Qb[B // 2:] ** 1.5
    got = ctx.significance_batch(dev(Pb), dev(Qb))
    for b in (0, 1, 255, 256, 511):
        S_o, lp_o, num_o = O.significance(Pb[b], Qb[b])
        assert got[b].stat.num == num_o
        assert abs(got[b].log_prod - lp_o) <= got[b].cells * tol_entry(50, 50) + 1e-12 * abs(lp_o)
    assert all(0.0 <= g.S <= 1.0 for g in got)


def test_significance_hand_derived_golden(ctx):
    # the GPU path against the hand-derived values of tests/golden/significance_hand.json (pinned for the
    # oracle in test_oracle_pins.py): integers exact, log_prod / S within the derived per-cell tolerance
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "significance_hand.json")))
    for c in g["cases"]:
        P, Q = np.array(c["P"], np.float32), np.array(c["Q"], np.float32)
        r = ctx.significance(dev(P), dev(Q))
        tol = sum(c["cells"].values()) * tol_entry(P.shape[0], Q.shape[0])
        assert (r.stat.num, r.stat.den) == (c["num"], c["den"]), c["name"]
        assert r.cells == sum(c["cells"].values())
        assert abs(r.log_prod - c["log_prod_value"]) <= tol, (c["name"], r.log_prod)
        assert abs(r.S - c["S_value"]) <= tol, (c["name"], r.S)
        if "poisson" in c:
            rp = ctx.significance(dev(P), dev(Q), poisson=True)
            assert abs(rp.log_prod - c["poisson"]["log_prod_value"]) <= tol, (c["name"], rp.log_prod)
