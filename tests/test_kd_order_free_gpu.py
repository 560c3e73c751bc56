"""The kd-ordered count must not depend on the row order (every per-tile / per-warp decision is taken from the actual
min / max of the rows involved): DDKS_KD_SHUFFLE scrambles the rows inside each label run after the kd sort, which
makes most boxes wide (few decided bits) and the order arbitrary; the statistic, argmax and the significance
histogram must equal the unscrambled and the position-ordered results."""
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


@pytest.mark.parametrize("shuffle", ["7", "40503", "1000003"])
@pytest.mark.parametrize("d,kind,n_P,n_Q,kd", [(2, "grid", 9000, 7000, "2,3,1"), (3, "normal", 20000, 18000, "3,3,3"),
                                               (5, "mixed", 30000, 26000, "4,3,2,2"), (5, "dup", 50000, 50001, None),
                                               (8, "mixed", 50000, 50001, None), (6, "grid", 12000, 9000, "4,2,2,2")])
def test_kd_counts_are_order_free(monkeypatch, shuffle, d, kind, n_P, n_Q, kd):
    P, Q = I.random_pair(4300 + d, n_P, n_Q, d, kind)
    if kind == "grid":
        P[:, : min(d, 4)] = np.round(P[:, : min(d, 4)] * 3) / 3
    if kd:
        monkeypatch.setenv("DDKS_KD", kd)
    with K.Context(flags=K.DDKS_FLAG_NO_X0 | K.DDKS_FLAG_NO_GRAPH) as pos:
        want = pos.stat(dev(P), dev(Q))
    with K.Context(flags=K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_NO_GRAPH) as c:
        assert c.stat(dev(P), dev(Q)) == want
        monkeypatch.setenv("DDKS_KD_SHUFFLE", shuffle)
        assert c.stat(dev(P), dev(Q)) == want
        assert c.kd_levels >= 1
