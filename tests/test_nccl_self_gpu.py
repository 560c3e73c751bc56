"""The multi-GPU collectives on one device: DDKS_FLAG_NCCL_SELF creates a one-rank NCCL communicator, so every
all-reduce / all-gather of the sharded paths (statistic, batch, permutation null, significance, vdKS, rdKS) runs
through NCCL with the real datatypes, counts, buffers and streams. Results must equal the plain single-rank path
(which skips the collectives). The rank > 1 combine logic itself is covered by tests/test_multirank_gloo.py."""
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
def pair():
    with K.Context() as plain, K.Context(flags=K.DDKS_FLAG_NCCL_SELF) as nccl:
        yield plain, nccl


@pytest.mark.parametrize("n,d,fl", [(3000, 3, 0), (150000, 5, 0), (20000, 4, K.DDKS_FLAG_FORCE_X0)])
def test_nccl_self_stat(pair, n, d, fl):
    P, Q = I.random_pair(300 + d, n, n - 7, d, "mixed")
    with K.Context(flags=fl) as a, K.Context(flags=fl | K.DDKS_FLAG_NCCL_SELF) as b:
        assert a.stat(dev(P), dev(Q)) == b.stat(dev(P), dev(Q))
        assert a.significance(dev(P), dev(Q)) == b.significance(dev(P), dev(Q))


def test_nccl_self_batch_perm_sig_batch(pair):
    plain, nccl = pair
    Pb, Qb = I.random_pair(31, 40 * 300, 40 * 280, 3, "normal")
    Pb, Qb = Pb.reshape(40, 300, 3), Qb.reshape(40, 280, 3)
    assert [r.num for r in plain.stat_batch(dev(Pb), dev(Qb))] == [r.num for r in nccl.stat_batch(dev(Pb), dev(Qb))]
    a = plain.significance_batch(dev(Pb[:, :50]), dev(Qb[:, :40]), poisson=True)
    b = nccl.significance_batch(dev(Pb[:, :50]), dev(Qb[:, :40]), poisson=True)
    assert a == b
    pooled = np.concatenate([Pb[0], Qb[0]])
    rng = np.random.default_rng(5)
    perms = np.stack([rng.permutation(580) for _ in range(37)]).astype(np.int32)
    for fl in (0, K.DDKS_FLAG_PERM_GATHER):
        with K.Context(flags=fl) as c1, K.Context(flags=fl | K.DDKS_FLAG_NCCL_SELF) as c2:
            n1, o1, p1 = c1.permutation_null(dev(pooled), 300, dev(perms))
            n2, o2, p2 = c2.permutation_null(dev(pooled), 300, dev(perms))
            assert np.array_equal(n1, n2) and o1 == o2 and p1 == p2


def test_nccl_self_approximations(pair):
    plain, nccl = pair
    P, Q = I.random_pair(41, 20000, 18000, 4, "normal")
    assert plain.vdks(dev(P), dev(Q), 8) == nccl.vdks(dev(P), dev(Q), 8)
    assert plain.rdks(dev(P), dev(Q)) == nccl.rdks(dev(P), dev(Q))
    s1 = plain.significance(dev(P[:300]), dev(Q[:200]), detail=True)
    s2 = nccl.significance(dev(P[:300]), dev(Q[:200]), detail=True)
    assert s1.stat == s2.stat and s1.log_prod == s2.log_prod and np.array_equal(s1.log_p_table, s2.log_p_table)
