"""Seeded fuzz of every GPU path against the oracle at sizes that straddle the kernels' internal boundaries: tile
sizes (256/512 points), the int16 flush window (32767 points), origin blocks (R*T), radix tiles (4096 keys), warp
and CTA edges, plus degenerate shapes (single points, one-sided samples, constant or duplicated coordinates)."""
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

SIZES = [1, 2, 31, 32, 33, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 3071, 3072, 3073, 4095, 4096, 4097]
KINDS = ["normal", "grid", "mixed", "dup"]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cases(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        n_P = int(rng.choice(SIZES))
        n_Q = int(rng.choice(SIZES))
        d = int(rng.integers(1, 9))
        out.append((n_P, n_Q, d, str(rng.choice(KINDS)), int(rng.integers(0, 2**31))))
    return out


@pytest.fixture(scope="module")
def ctxs():
    cs = {name: K.Context(flags=f) for name, f in [("default", 0), ("x0", K.DDKS_FLAG_FORCE_X0),
                                                    ("direct", K.DDKS_FLAG_FORCE_DIRECT),
                                                    ("x0gt", K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_TIES_GT),
                                                    ("full", K.DDKS_FLAG_RDKS_FULL_SORT),
                                                    ("kd2", K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(2)),
                                                    ("kd3", K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(3)),
                                                    ("kd4", K.DDKS_FLAG_FORCE_X0)]}
    yield cs
    for c in cs.values():
        c.close()


@pytest.mark.parametrize("n_P,n_Q,d,kind,seed", cases(2024, int(os.environ.get("DDKS_FUZZ_CASES", "36"))))
def test_fuzz_exact_and_approx(monkeypatch, ctxs, n_P, n_Q, d, kind, seed):
    P, Q = I.random_pair(seed, n_P, n_Q, d, kind)
    want = O.ddks(P, Q)
    for name in ("default", "x0", "direct"):
        r = ctxs[name].stat(dev(P), dev(Q))
        assert (r.num, r.den, r.argmax_origin) == (want[0], want[1], want[3]), name
    # kd levels 2, 3 and 4 (capped at d) with seeded slab / cell counts (many empty or single-tile cells at these sizes)
    for K_ in (2, 3, 4):
        monkeypatch.setenv("DDKS_KD", f"{K_},{1 + seed % 6},{1 + (seed // 6) % 5},{1 + (seed // 30) % 4}")
        r = ctxs[f"kd{K_}"].stat(dev(P), dev(Q))
        assert (r.num, r.den, r.argmax_origin) == (want[0], want[1], want[3]), (K_, os.environ["DDKS_KD"])
    monkeypatch.delenv("DDKS_KD")
    gt = O.ddks(P, Q, ties_gt=True)
    r = ctxs["x0gt"].stat(dev(P), dev(Q))
    assert (r.num, r.argmax_origin) == (gt[0], gt[3])
    k = 2 + seed % 5
    if k ** d <= 1 << 16:
        assert ctxs["default"].vdks(dev(P), dev(Q), k)[:2] == O.vdks(P, Q, k)[:2]
    rd = O.rdks(P, Q)
    for name in ("default", "full"):
        r = ctxs[name].rdks(dev(P), dev(Q))
        assert (r.num, r.argmax_origin) == (rd[0], rd[3]), name


@pytest.mark.parametrize("n,d,kind,seed", [(32767, 2, "grid", 1), (32768, 3, "normal", 2), (40001, 5, "dup", 3),
                                           (65535, 1, "grid", 4)])
def test_fuzz_flush_window_edges(ctxs, n, d, kind, seed):
    # pooled sizes at the int16 flush window and the 16-bit permutation-counter limit
    P, Q = I.random_pair(seed, n // 2, n - n // 2, d, kind)
    want = O.ddks(P, Q)
    for name in ("default", "x0"):
        r = ctxs[name].stat(dev(P), dev(Q))
        assert (r.num, r.argmax_origin) == (want[0], want[3]), name


@pytest.mark.parametrize("n_P,n_Q,d,n_perm,seed", [(1, 1, 2, 3, 5), (257, 255, 3, 17, 6), (511, 513, 5, 33, 7),
                                                   (1000, 24, 8, 9, 8)])
def test_fuzz_batch_and_permutations(ctxs, n_P, n_Q, d, n_perm, seed):
    rng = np.random.default_rng(seed)
    B = 7
    Pb = rng.standard_normal((B, n_P, d)).astype(np.float32)
    Qb = np.round(rng.standard_normal((B, n_Q, d)) * 2).astype(np.float32)
    got = ctxs["default"].stat_batch(dev(Pb), dev(Qb))
    assert np.array_equal(got.num, O.batch(Pb, Qb))
    pooled = np.concatenate([Pb[0], Qb[0]])
    N = n_P + n_Q
    perms = np.stack([rng.permutation(N) for _ in range(n_perm)]).astype(np.int32)
    null, obs, p = ctxs["default"].permutation_null(dev(pooled), n_P, dev(perms))
    o_null, o_obs, _, o_p = O.permutation_null(pooled, n_P, perms)
    assert np.array_equal(null, o_null) and obs.num == o_obs and p == o_p
