"""Pins of the CPU oracle against things other than itself (PAPER.md / SPEC.md examples, closed forms,
invariants, brute force). No GPU. Each test names the passage it follows; see DESIGN.md "Oracle pins".

A plausible mistake anywhere in the oracle fails at least one of these:
  * dropped Q (or P) counts, or a dropped origin self-count   -> SPEC examples, tie example, 1-D KS
  * '>' instead of '>='                                       -> tie example, C3 cross-check
  * wrong sign / wrong normalisation / swapped n_P, n_Q        -> unequal-size example, 1-D KS, replication
  * transposed operand (origin vs point)                      -> SPEC membership/orthant examples, line embedding
  * bit order / orthant index mixups                          -> SPEC orthant_index examples, membership
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.stats

from oracle import oracle as O
from paper_2106_13706_b200 import inputs as I


def _frac(num, den):
    return Fraction(num, den)


# ------------------------------------------------------------------------------------ SPEC examples

def test_spec_orthant_index(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["orthant_index"]:
        assert O.orthant_index(c["test"], c["point"]) == c["expect"], c["cite"]


def test_spec_membership(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["membership"]:
        got = O.membership(np.array(c["counted"], np.float32), np.array(c["test"], np.float32))
        assert got.tolist() == c["expect"], c["cite"]


def test_spec_statistic(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["statistic"]:
        num, den, D, _ = O.ddks(np.array(c["P"], np.float32), np.array(c["Q"], np.float32))
        assert _frac(num, den) == Fraction(c["D_num"], c["D_den"]), c["cite"]
        assert O.brute_force(c["P"], c["Q"]) == Fraction(c["D_num"], c["D_den"]), c["cite"]


def test_hand_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "hand_examples.json")))
    for c in g["cases"]:
        P, Q = np.array(c["P"], np.float32), np.array(c["Q"], np.float32)
        num, den, D, _ = O.ddks(P, Q)
        assert (num, den) == (c["ge"]["num"], c["ge"]["den"]), c["name"]
        assert D == num / den
        assert O.brute_force(P, Q) == Fraction(c["ge"]["num"], c["ge"]["den"]), c["name"]
        if "gt" in c:
            num, den, _, _ = O.ddks(P, Q, ties_gt=True)
            assert (num, den) == (c["gt"]["num"], c["gt"]["den"]), c["name"]
            assert O.brute_force(P, Q, ties_gt=True) == Fraction(c["gt"]["num"], c["gt"]["den"])


def test_membership_rows_sum_to_n():
    # SPEC S:L113 / S:L94-97: each counted point falls in exactly one orthant per test point.
    P, Q = I.random_pair(11, 37, 23, 4, "grid")
    M = O.membership(P, Q)
    assert M.shape == (23, 16)
    assert (M.sum(axis=1) == 37).all()
    # the test point itself (as a counted point) lands in the all-ones orthant (>= on every axis)
    M2 = O.membership(Q, Q)
    assert (M2[:, 15] >= 1).all()


# ------------------------------------------------------------------------------------ brute force

@pytest.mark.parametrize("ties_gt", [False, True])
def test_oracle_equals_brute_force_tiny(ties_gt):
    # exhaustive-style random tiny inputs, integer grid 0..3 so ties dominate (SURVEY.md §8c "Brute force")
    rng = np.random.default_rng(1234)
    for trial in range(150):
        d = int(rng.integers(1, 5))
        n_P = int(rng.integers(1, 8))
        n_Q = int(rng.integers(1, 8))
        kind = ["grid", "normal", "mixed"][trial % 3]
        P, Q = I.random_pair(10_000 + trial, n_P, n_Q, d, kind)
        num, den, D, _ = O.ddks(P, Q, ties_gt=ties_gt)
        assert den == n_P * n_Q
        assert Fraction(num, den) == O.brute_force(P, Q, ties_gt=ties_gt), (trial, d, n_P, n_Q, kind)


# ------------------------------------------------------------------------------------ closed forms

def test_one_dimensional_equals_classical_ks():
    # d = 1: ddKS is the two-sample KS statistic (derivation DESIGN.md "Oracle pins" #4)
    rng = np.random.default_rng(7)
    for trial in range(200):
        n_P, n_Q = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        if trial % 2:
            u_P, u_Q = rng.integers(0, 6, n_P).astype(np.float32), rng.integers(0, 6, n_Q).astype(np.float32)
        else:
            u_P, u_Q = rng.standard_normal(n_P).astype(np.float32), (rng.standard_normal(n_Q) + 0.3).astype(np.float32)
        num, den, D, _ = O.ddks(u_P[:, None], u_Q[:, None])
        ks_num, ks_den = O.ks_1d(u_P, u_Q)
        assert (num, den) == (ks_num, ks_den), trial
        assert abs(D - float(scipy.stats.ks_2samp(u_P.astype(np.float64), u_Q.astype(np.float64)).statistic)) <= 1e-12, trial


def test_diagonal_embedding_equals_1d_ks():
    # every point x = u * (1,...,1): all coordinates tie together, so ddKS = 1-D KS of u (P:L322 DVU diagonal)
    rng = np.random.default_rng(8)
    for trial in range(60):
        d = int(rng.integers(2, 9))
        u_P = rng.integers(0, 8, int(rng.integers(1, 40))).astype(np.float32)
        u_Q = rng.integers(0, 8, int(rng.integers(1, 40))).astype(np.float32)
        P = np.repeat(u_P[:, None], d, axis=1)
        Q = np.repeat(u_Q[:, None], d, axis=1)
        num, den, _, _ = O.ddks(P, Q)
        assert (num, den) == O.ks_1d(u_P, u_Q), trial


def test_mixed_sign_line_embedding():
    # x = u * s, s in {+-1}^d with both signs: three orthants about every origin (u>v, u<v, u=v), so
    # num = max(KS_num(u_P, u_Q), max_v |m_P(v) n_Q - m_Q(v) n_P|)   (DESIGN.md "Oracle pins" #6)
    rng = np.random.default_rng(9)
    for trial in range(80):
        d = int(rng.integers(2, 6))
        s = np.ones(d, np.float32)
        neg = rng.choice(d, size=int(rng.integers(1, d)), replace=False)
        s[neg] = -1.0
        u_P = rng.integers(-4, 5, int(rng.integers(1, 30))).astype(np.float32)
        u_Q = rng.integers(-4, 5, int(rng.integers(1, 30))).astype(np.float32)
        P, Q = u_P[:, None] * s[None, :], u_Q[:, None] * s[None, :]
        n_P, n_Q = len(u_P), len(u_Q)
        ks_num, _ = O.ks_1d(u_P, u_Q)
        mass = max(abs(int((u_P == v).sum()) * n_Q - int((u_Q == v).sum()) * n_P) for v in np.concatenate([u_P, u_Q]))
        num, den, _, _ = O.ddks(P, Q)
        assert num == max(ks_num, mass), trial
        assert den == n_P * n_Q


def test_constant_coordinate_reduces_dimension():
    # a coordinate equal for every point is always a tie (bit set), so it drops out
    for seed in range(20):
        P, Q = I.random_pair(seed, 17, 13, 3, "mixed")
        c = np.float32(0.625)
        P4 = np.concatenate([P, np.full((17, 1), c, np.float32)], axis=1)
        Q4 = np.concatenate([np.full((13, 1), c, np.float32), Q], axis=1)[:, [1, 2, 3, 0]]
        assert O.ddks(P4, Q4)[:2] == O.ddks(P, Q)[:2]


def test_full_separation_gives_one():
    # max_P x_k < min_Q x_k for every k => D = 1 (at the Q origin minimising x_0: all P in orthant 0, no Q)
    rng = np.random.default_rng(10)
    for trial in range(30):
        d = int(rng.integers(1, 6))
        P = rng.random((int(rng.integers(1, 30)), d)).astype(np.float32)
        Q = (rng.random((int(rng.integers(1, 30)), d)) + 1.5).astype(np.float32)
        num, den, D, _ = O.ddks(P, Q)
        assert num == den and D == 1.0


# ------------------------------------------------------------------------------------ invariants (App. A)

def test_identity_symmetry_range():
    rng = np.random.default_rng(11)
    for trial in range(40):
        d = int(rng.integers(1, 6))
        kind = ["grid", "normal", "dup", "mixed"][trial % 4]
        P, Q = I.random_pair(500 + trial, int(rng.integers(1, 40)), int(rng.integers(1, 40)), d, kind)
        assert O.ddks(P, P)[0] == 0                                   # P:L458-465 identity
        a = O.ddks(P, Q)
        b = O.ddks(Q, P)
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]          # P:L467-469 symmetry (exact)
        assert 0 <= a[0] <= a[1]                                       # SPEC S:L144 range


def test_exact_invariances():
    # row shuffle, axis permutation, power-of-two scaling, dense-rank (strictly increasing) map
    rng = np.random.default_rng(12)
    for trial in range(30):
        d = int(rng.integers(1, 6))
        P, Q = I.random_pair(900 + trial, int(rng.integers(2, 40)), int(rng.integers(2, 40)), d,
                             ["normal", "grid", "mixed"][trial % 3])
        ref = O.ddks(P, Q)[:2]
        assert O.ddks(P[rng.permutation(len(P))], Q[rng.permutation(len(Q))])[:2] == ref
        ax = rng.permutation(d)
        assert O.ddks(P[:, ax], Q[:, ax])[:2] == ref
        assert O.ddks(P * np.float32(8.0), Q * np.float32(8.0))[:2] == ref
        pooled = np.concatenate([P, Q])
        R = np.empty_like(pooled)
        for k in range(d):
            R[:, k] = np.searchsorted(np.unique(pooled[:, k]), pooled[:, k]).astype(np.float32)
        assert O.ddks(R[: len(P)], R[len(P):])[:2] == ref


def test_negation_is_not_an_invariance():
    # DESIGN.md reading R11: decreasing maps move ties to the other side; the tie example shows it
    P, Q = np.array([[2, 1]], np.float32), np.array([[1, 1], [2, 0]], np.float32)
    assert O.ddks(P, Q)[:2] != O.ddks(-P, -Q)[:2]


def test_replication_invariance():
    # a copies of P and b copies of Q: counts scale, origin values unchanged -> num*a*b, den*a*b, same D
    rng = np.random.default_rng(13)
    for trial in range(25):
        d = int(rng.integers(1, 5))
        P, Q = I.random_pair(1300 + trial, int(rng.integers(1, 15)), int(rng.integers(1, 15)), d, "grid")
        a, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        num, den, D, _ = O.ddks(P, Q)
        num2, den2, D2, _ = O.ddks(np.tile(P, (a, 1)), np.tile(Q, (b, 1)))
        assert (num2, den2) == (num * a * b, den * a * b) and D2 == D


# ------------------------------------------------------------------------------------ batch / permutations

def test_batch_and_permutation_consistency():
    rng = np.random.default_rng(14)
    B, n_P, n_Q, d = 5, 9, 7, 3
    P = rng.integers(0, 4, (B, n_P, d)).astype(np.float32)
    Q = rng.integers(0, 4, (B, n_Q, d)).astype(np.float32)
    got = O.batch(P, Q)
    for b in range(B):
        assert got[b] == O.ddks(P[b], Q[b])[0]
    pooled = np.concatenate([P[0], Q[0]])
    perms = np.stack([np.arange(n_P + n_Q)] + [rng.permutation(n_P + n_Q) for _ in range(20)]).astype(np.int32)
    null, obs, p_num, p = O.permutation_null(pooled, n_P, perms)
    assert obs == O.ddks(P[0], Q[0])[0]
    assert null[0] == obs                                             # identity permutation = observed
    for j in range(1, len(perms)):
        assert null[j] == O.ddks(pooled[perms[j][:n_P]], pooled[perms[j][n_P:]])[0]
    assert p_num == 1 + int((null >= obs).sum()) and p == p_num / (1 + len(perms))


def test_permutation_disjoint_clusters_pvalue():
    # disjoint 1-D clusters, observed D = 1 beats (almost) every relabelling
    rng = np.random.default_rng(15)
    P = rng.random((20, 1)).astype(np.float32)
    Q = (rng.random((20, 1)) + 2).astype(np.float32)
    perms = np.stack([rng.permutation(40) for _ in range(100)]).astype(np.int32)
    null, obs, p_num, p = O.permutation_null(np.concatenate([P, Q]), 20, perms)
    assert obs == 400 and p_num == 1 and p == 1 / 101


# ------------------------------------------------------------------------------------ configs (inputs + cross-check)

@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_config_inputs_match_survey_bytes(name):
    P, Q = I.config(name)
    assert I.sha256_pq(P, Q) == I.SURVEY_SHA256[name]


def test_c1_c2_values_match_independent_survey_computation():
    # SURVEY.md §8c "Survey-time reference values": an independent vectorised NumPy exact-integer implementation,
    # valid because our input bytes match (test above). C1: 6000/40000 at origin 124; C2: 6,760,000/1e8 at 11,829.
    P, Q = I.config("C1")
    assert O.ddks(P, Q) == (6000, 40000, 0.15, 124)
    assert O.ddks(P, Q, ties_gt=True)[0] == 6000
    assert O.ddks(Q, P)[0] == 6000
    P, Q = I.config("C2")
    num, den, D, arg = O.ddks(P, Q)
    assert (num, den, arg) == (6_760_000, 100_000_000, 11_829)
    assert D.hex() == "0x1.14e3bcd35a858p-4"


@pytest.mark.slow
def test_c3_tie_convention_changes_result():
    # C3 num 15,320,000 (>=) vs 15,340,000 (>), argmax origin 27,347
    P, Q = I.config("C3")
    num, den, D, arg = O.ddks(P, Q)
    assert (num, den, arg) == (15_320_000, 400_000_000, 27_347)
    assert D.hex() == "0x1.39c0ebedfa440p-5"
    assert O.ddks(P, Q, ties_gt=True)[0] == 15_340_000


@pytest.mark.slow
def test_c5_per_origin_spots():
    # SURVEY.md §8c C5 per-origin spot values (num(o) in units of 1e6; > 2^32 so 64-bit is required)
    P, Q = I.config("C5")
    spots = {0: 27017, 1: 37275, 2: 17948, 3: 42316, 999999: 20278, 1000000: 32904, 1000001: 14470,
             1999999: 14910, 123456: 15831, 1765432: 38497}
    for o, v in spots.items():
        assert int(O.per_origin(P, Q, o, o + 1)[0]) == v * 1_000_000, o
    assert int(O.per_origin(P, Q, 1, 2, ties_gt=True)[0]) == 37276 * 1_000_000


@pytest.mark.slow
def test_c4_spots():
    # SURVEY.md §8c C4a per-pair nums and C4b permutation null on pair 2048
    P, Q = I.config("C4")
    idx = [0, 1, 2, 3, 4, 2048, 2049, 2050, 2051, 2052]
    want = [19968, 19456, 31232, 24576, 19456, 39936, 36352, 30208, 39424, 30720]
    got = O.batch(P[idx], Q[idx])
    assert got.tolist() == want
    perms = I.c4_perms()
    pooled = np.concatenate([P[I.C4_PERM_PAIR], Q[I.C4_PERM_PAIR]])
    null, obs, p_num, p = O.permutation_null(pooled, 512, perms)
    assert obs == 39936 and int(null.max()) == 34816 and int(null.sum()) == 23_215_616
    assert p_num == 1 and p == 1 / 1001


def test_stored_c4_oracle_matches_survey_aggregates(golden_dir):
    # tests/golden/c4_oracle.json (every C4a item, every C4b permutation; written by make_c4_oracle.py, oracle only)
    # belongs to these input bytes and this oracle source, and agrees with the survey's independent NumPy computation
    # (SURVEY.md §8c C4a/C4b rows): the per-pair spots, the max and the sum over all 4096 items, the null's max and sum
    import hashlib
    g = json.load(open(os.path.join(golden_dir, "c4_oracle.json")))
    assert g["input_sha256"] == I.SURVEY_SHA256["C4"] and g["perms_sha256"] == I.SURVEY_SHA256["C4_perms"]
    src = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "ddks_oracle.c"), "rb").read()
    assert g["oracle_c_sha256"] == hashlib.sha256(src).hexdigest()
    b = np.array(g["batch_num"], dtype=np.int64)
    assert len(b) == 4096 and g["den"] == 512 * 512
    assert b[:5].tolist() == [19968, 19456, 31232, 24576, 19456]
    assert b[2048:2053].tolist() == [39936, 36352, 30208, 39424, 30720]
    assert int(b.max()) == 56_320 and int(b.sum()) == 122_770_432
    null = np.array(g["null_num"], dtype=np.int64)
    assert len(null) == 1000 and int(null.max()) == 34_816 and int(null.sum()) == 23_215_616
    assert g["observed_num"] == 39_936 == b[2048] and g["p_num"] == 1 and g["p_value"] == 1 / 1001


# ------------------------------------------------------------------------------------ analytic significance (§3)

def test_significance_pmf_pins():
    import scipy.stats as st
    # SPEC S:L330-332 binomial_pmf examples and the zero-success closed form
    assert abs(math.exp(O.log_pmf(1, 2, 0.5)) - 0.5) < 1e-15
    for m, lam in [(7, 0.3), (50, 0.02), (1000, 0.5)]:
        assert abs(math.exp(O.log_pmf(0, m, lam)) - (1 - lam) ** m) <= 1e-12 * max((1 - lam) ** m, 1e-300)
        tot = sum(math.exp(O.log_pmf(n, m, lam)) for n in range(m + 1))
        assert abs(tot - 1.0) < 1e-10
        # textbook pmfs (binomial, Poisson) from an independent library implementation
        for n in (0, 1, m // 3, m):
            assert abs(math.exp(O.log_pmf(n, m, lam)) - st.binom.pmf(n, m, lam)) <= 1e-11 * max(st.binom.pmf(n, m, lam), 1e-300) + 1e-300
            assert abs(math.exp(O.log_pmf(n, m, lam, poisson=True)) - st.poisson.pmf(n, m * lam)) <= 1e-11 * max(st.poisson.pmf(n, m * lam), 1e-300) + 1e-300


def test_significance_p_le_pins():
    # SPEC S:L340-342 delta_cdf four-outcome enumerations (n_p = n_t = 1, lambda = 0.5)
    assert abs(O.p_le(0, 1, 1, 0.5) - 0.5) < 1e-15        # D = 0: (0,0) and (1,1)
    assert abs(O.p_le(1, 1, 1, 0.5) - 1.0) < 1e-15        # D = 1: everything
    for lam in (0.1, 0.37, 0.9):                            # closed form P(X = Y), X, Y ~ Bernoulli(lam)
        assert abs(O.p_le(0, 1, 1, lam) - (lam * lam + (1 - lam) ** 2)) < 1e-14
    # D = 1 covers the whole Delta-set: the factor is 1 (sum of all pmf products)
    assert abs(O.p_le(30 * 40, 30, 40, 0.23) - 1.0) < 1e-12
    # monotone in D; symmetric under lambda -> 1 - lambda when N_P = N_T (n -> N - n maps the band to itself)
    vals = [O.p_le(num, 20, 20, 0.3) for num in range(0, 401, 20)]
    assert all(b >= a - 1e-15 for a, b in zip(vals, vals[1:]))
    assert abs(O.p_le(60, 20, 20, 0.3) - O.p_le(60, 20, 20, 0.7)) < 1e-13


def test_significance_p_le_against_monte_carlo():
    # an independent estimate of P(|X/N_P - Y/N_T| <= D), X ~ Bi(N_P, l), Y ~ Bi(N_T, l): within 5 sigma
    rng = np.random.default_rng(31)
    for (N_P, N_T, lam, num) in [(12, 9, 0.3, 20), (50, 50, 0.05, 150), (40, 25, 0.6, 60)]:
        n = 400_000
        X = rng.binomial(N_P, lam, n)
        Y = rng.binomial(N_T, lam, n)
        frac = np.mean(np.abs(X * N_T - Y * N_P) <= num)
        p = O.p_le(num, N_P, N_T, lam)
        assert abs(frac - p) <= 5 * math.sqrt(p * (1 - p) / n) + 1e-9, (N_P, N_T, lam, num, frac, p)


def test_significance_statistic_pins():
    # fully separated samples: D = 1, every factor is 1 -> S = 0
    rng = np.random.default_rng(32)
    P = rng.random((12, 2)).astype(np.float32)
    Q = (rng.random((10, 2)) + 2).astype(np.float32)
    S, lp, num = O.significance(P, Q)
    assert num == 120 and abs(S) < 1e-12
    # identical samples: D = 0, cannot reject (S > 0.9)
    P = rng.random((50, 3)).astype(np.float32)
    S, lp, num = O.significance(P, P.copy())
    assert num == 0 and S > 0.9
    # S is a probability; Poisson variant close to binomial when rates are small
    P, Q = I.random_pair(33, 40, 30, 3, "normal")
    S_b, _, _ = O.significance(P, Q)
    S_p, _, _ = O.significance(P, Q, poisson=True)
    assert 0.0 <= S_b <= 1.0 and 0.0 <= S_p <= 1.0


def test_significance_hand_derived_golden(golden_dir):
    # tests/golden/significance_hand.json: S derived by hand from P:L208-209 (test points = both sets)
    # (lambda-hat = (M_T+1)/(N_T+2)), P:L244-268 (binomial pmf, Delta band), P:L276 (product over all 2^d x N cells,
    # empty orthants included) and P:L278-281 (Poisson). The alternative readings (lambda = M_T/N_T; T-only test
    # points) give values far outside the tolerance, so either mistake fails here.
    g = json.load(open(os.path.join(golden_dir, "significance_hand.json")))
    for c in g["cases"]:
        P, Q = np.array(c["P"], np.float32), np.array(c["Q"], np.float32)
        S, lp, num = O.significance(P, Q)
        assert num == c["num"] and P.shape[0] * Q.shape[0] == c["den"], c["name"]
        assert abs(lp - c["log_prod_value"]) <= 1e-14, (c["name"], lp)
        assert abs(S - c["S_value"]) <= 1e-14, (c["name"], S)
        for reading, alt in c.get("other_readings", {}).items():
            assert abs(alt["log_prod_value"] - c["log_prod_value"]) > 0.1, reading
        if "poisson" in c:
            _, lpp, _ = O.significance(P, Q, poisson=True)
            assert abs(lpp - c["poisson"]["log_prod_value"]) <= 1e-14, (c["name"], lpp)
        # the factors themselves: p(d <= D | lambda-hat) per M_T value
        for key, frac in c["factors"].items():
            m = int(key.split("=")[1])
            lam = (m + 1) / (Q.shape[0] + 2)
            assert abs(O.p_le(c["num"], P.shape[0], Q.shape[0], lam) - float(Fraction(frac))) <= 1e-15, (c["name"], key)


# ------------------------------------------------------------------------------------ vdKS (Alg. 1) and rdKS (Alg. 2)

def _grid_pair(seed, n_P, n_Q, d, k):
    """Integer-grid samples whose every coordinate takes values 0..k-1 with both ends present in every dimension
    (so NormalizeData maps value v to v/(k-1) and Alg. 1's floor(x' k), clamped, is cell v)."""
    rng = np.random.default_rng(seed)
    P = rng.integers(0, k, (n_P, d)).astype(np.float32)
    Q = rng.integers(0, k, (n_Q, d)).astype(np.float32)
    P[0, :], Q[0, :] = 0, k - 1
    return P, Q


def test_spec_voxel_and_sweep_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["voxel_index"]:
        assert O.voxel_index(c["point"], c["k"]) == c["expect"], c["cite"]
    for c in g["vdks"]:
        num, den, D = O.vdks(np.array(c["P"], np.float32), np.array(c["Q"], np.float32), c["k"])
        assert Fraction(num, den) == Fraction(c["D_num"], c["D_den"]), c["cite"]
    for c in g["merged_max_diff"]:
        num = O.merged_max_diff(c["a"], c["b"])
        assert Fraction(num, len(c["a"]) * len(c["b"])) == Fraction(c["D_num"], c["D_den"]), c["cite"]
    for c in g["normalize"]:
        got = O.normalize_pair(np.array(c["P"], np.float32), np.array(c["Q"], np.float32))
        assert got.tolist() == c["expect"], c["cite"]


def test_vdks_is_exact_ddks_on_cells():
    # Alg. 1's orthant sums about a filled voxel's lower corner (the voxel itself in the all->= orthant) are the
    # exact ddKS orthant counts of the cell-index points; the filled voxels are the distinct origins. On an
    # integer grid 0..k-1 whose ends are present, cell = value, so vdKS(k) == exact ddKS (an independent oracle).
    for seed, (n_P, n_Q, d, k) in enumerate([(30, 20, 1, 5), (40, 33, 2, 4), (25, 31, 3, 3), (60, 50, 3, 6),
                                              (20, 24, 4, 3), (12, 15, 5, 2)]):
        P, Q = _grid_pair(seed, n_P, n_Q, d, k)
        assert O.vdks(P, Q, k)[:2] == O.ddks(P, Q)[:2], (n_P, n_Q, d, k)
        # the same holds after strictly increasing affine maps per coordinate (NormalizeData removes them)
        A = P * np.float32(4.0) - np.float32(3.0)
        B = Q * np.float32(4.0) - np.float32(3.0)
        assert O.vdks(A, B, k)[:2] == O.ddks(P, Q)[:2]


def test_vdks_properties():
    P, Q = I.random_pair(51, 90, 70, 3, "normal")
    assert O.vdks(P, Q, 1)[0] == 0                                  # one voxel: all orthant sums are 0 or total 0
    assert O.vdks(P, P.copy(), 7)[0] == 0                           # identity
    for k in (2, 5, 9):
        a, b = O.vdks(P, Q, k), O.vdks(Q, P, k)
        assert a[0] == b[0] and 0 <= a[0] <= a[1]                   # symmetry (|.|, R16), range
    # invariance under per-coordinate scaling by powers of two (exact in float32)
    s = np.array([2.0, 0.5, 8.0], np.float32)
    assert O.vdks(P * s, Q * s, 6) == O.vdks(P, Q, 6)
    # brute force on tiny inputs: the definition of SumOrthants as a Fraction over the cell points
    for seed in range(40):
        P, Q = _grid_pair(100 + seed, 3 + seed % 4, 2 + seed % 5, 1 + seed % 3, 2 + seed % 3)
        num, den, _ = O.vdks(P, Q, 2 + seed % 3)
        assert Fraction(num, den) == O.brute_force(P, Q)


def _normalised_dyadic(seed, n_P, n_Q, d):
    """Points on the grid {0, 1/4, ..., 1} with 0 and 1 present per dimension: NormalizeData is the identity and
    every squared distance to a corner is an exact dyadic sum (so any evaluation order gives the same doubles)."""
    rng = np.random.default_rng(seed)
    P = (rng.integers(0, 5, (n_P, d)) / 4).astype(np.float32)
    Q = (rng.integers(0, 5, (n_Q, d)) / 4).astype(np.float32)
    P[0, :], Q[0, :] = 0, 1
    return P, Q


def _rdks_brute(P, Q):
    """Definition: max over corners c and radii r of |#P(|x-c| <= r)/n_P - #Q(|x-c| <= r)/n_Q| (Fractions)."""
    d = P.shape[1]
    best = Fraction(0)
    for ci in range(d + 1):
        c = np.zeros(d)
        if ci:
            c[ci - 1] = 1.0
        dp = [math.sqrt(sum((float(x) - cc) ** 2 for x, cc in zip(row, c))) for row in P.astype(np.float64)]
        dq = [math.sqrt(sum((float(x) - cc) ** 2 for x, cc in zip(row, c))) for row in Q.astype(np.float64)]
        for r in dp + dq:
            v = abs(Fraction(sum(x <= r for x in dp), len(dp)) - Fraction(sum(x <= r for x in dq), len(dq)))
            best = max(best, v)
    return best


def test_rdks_pins():
    # d = 1: corner 0's distances are x' itself (sqrt(x'^2) == |x'| in IEEE arithmetic), so rdKS = the classical
    # two-sample KS (corner 1 can only merge values, never exceed it) — against the independently pinned ks_1d
    for seed in range(30):
        rng = np.random.default_rng(200 + seed)
        u = rng.standard_normal(40 + seed).astype(np.float32)
        v = (rng.standard_normal(35) + 0.3 * (seed % 3)).astype(np.float32)
        if seed % 2:
            u, v = np.round(u * 2).astype(np.float32), np.round(v * 2).astype(np.float32)
        num, den, _, _ = O.rdks(u[:, None], v[:, None])
        assert Fraction(num, den) == Fraction(*O.ks_1d(u, v)), seed
    # brute force on exact dyadic distances
    for seed in range(25):
        P, Q = _normalised_dyadic(300 + seed, 3 + seed % 6, 2 + seed % 5, 1 + seed % 4)
        num, den, _, _ = O.rdks(P, Q)
        assert Fraction(num, den) == _rdks_brute(P, Q), seed
    # identity, symmetry, range, invariance under per-coordinate scaling by powers of two
    P, Q = I.random_pair(61, 120, 90, 4, "normal")
    assert O.rdks(P, P.copy())[0] == 0
    a, b = O.rdks(P, Q), O.rdks(Q, P)
    assert a[0] == b[0] and 0 <= a[0] <= a[1]
    s = np.array([2.0, 0.25, 4.0, 1.0], np.float32)
    assert O.rdks(P * s, Q * s)[:2] == a[:2]


def test_stored_c5_oracle_matches_inputs_and_oracle_source():
    # the stored full-C5 oracle result (tests/golden/make_c5_oracle.py) belongs to these input bytes and this oracle
    import hashlib
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_oracle.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c5_oracle.json not generated yet")
    g = json.load(open(path))
    assert g["input_sha256"] == I.SURVEY_SHA256["C5"]
    src = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "ddks_oracle.c"), "rb").read()
    assert g["oracle_c_sha256"] == hashlib.sha256(src).hexdigest()
    assert g["den"] == 10**12 and 0 < g["num"] <= g["den"] and float.fromhex(g["D_hex"]) == g["num"] / g["den"]
    # the survey's independent per-origin spot values bound it from below
    assert g["num"] >= 42316 * 10**6


def test_stored_c5_vdks_oracle_matches_inputs_and_oracle_source(golden_dir):
    # tests/golden/c5_vdks16_oracle.json (make_c5_vdks_oracle.py, oracle only) belongs to these input bytes and this
    # oracle source; its own value is pinned by the vdKS pins above (vdKS(k) == exact ddKS of the cell points, affine
    # invariance, brute force), which test the same oracle function at small sizes
    import hashlib
    g = json.load(open(os.path.join(golden_dir, "c5_vdks16_oracle.json")))
    assert g["input_sha256"] == I.SURVEY_SHA256["C5"] and g["k"] == 16
    src = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "ddks_oracle.c"), "rb").read()
    assert g["oracle_c_sha256"] == hashlib.sha256(src).hexdigest()
    assert g["den"] == 10**12 and 0 < g["num"] <= g["den"] and float.fromhex(g["D_hex"]) == g["num"] / g["den"]
    assert g["num"] % 10**6 == 0  # n_P = n_Q: every |orthant sum| is a multiple of n_P (exact integer Diff, R16)
