"""The kd-ordered count at sizes where it is the production path (N >= 80000: several cells per level, many point
segments, per-warp decisions, strided shards), cross-checked against the position-ordered count (which the oracle pins
at smaller sizes, and the stored C5 oracle pins at full size) on tie-heavy and continuous data, d = 2..8."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def ctxs():
    # NO_RANK: these tests are about the kd-ordered FP32 count (the rank-lane count would take some of the sizes)
    with K.Context(flags=K.DDKS_FLAG_NO_RANK) as kd, K.Context(flags=K.DDKS_FLAG_NO_X0 | K.DDKS_FLAG_NO_RANK) as pos:
        yield kd, pos


@pytest.mark.parametrize("d,kind,n_P,n_Q", [(2, "grid", 90000, 70000), (3, "normal", 80000, 80000),
                                            (4, "dup", 100000, 60000), (5, "mixed", 120000, 120000),
                                            (6, "grid", 70000, 90000), (7, "normal", 60000, 61000),
                                            (8, "mixed", 50000, 50001)])
def test_kd_matches_position_order_at_scale(ctxs, d, kind, n_P, n_Q):
    kd, pos = ctxs
    P, Q = I.random_pair(4000 + d, n_P, n_Q, d, kind)
    if kind == "grid":
        P[:, : min(d, 4)] = np.round(P[:, : min(d, 4)] * 4) / 4  # ties on every sorted dim
    a = kd.stat(dev(P), dev(Q))
    assert kd.kd_levels >= 1
    b = pos.stat(dev(P), dev(Q))
    assert a == b
    # every rank's strided kd shard combines to the same statistic
    for world in (3, 8):
        parts = [kd.stat_shard(dev(P), dev(Q), world, r) for r in range(world)]
        num = max(p.num for p in parts)
        assert num == a.num and min(p.argmax_origin for p in parts if p.num == num) == a.argmax_origin


def test_kd_significance_matches_position_order_at_scale(ctxs):
    kd, pos = ctxs
    P, Q = I.random_pair(4100, 60000, 45000, 5, "mixed")
    a = kd.significance(dev(P), dev(Q), detail=True)
    assert kd.kd_levels >= 1
    b = pos.significance(dev(P), dev(Q), detail=True)
    assert a.stat == b.stat and np.array_equal(a.mt_hist, b.mt_hist) and a.log_prod == b.log_prod
