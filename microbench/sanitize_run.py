"""Small invocation of every library path, for compute-sanitizer (memcheck / racecheck / synccheck).
Each result is checked against the oracle so a sanitizer run also proves the instrumented kernels still agree."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2106_13706_b200 import ddks as K, inputs as I


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


P, Q = I.random_pair(3, 700, 650, 3, "mixed")
want = O.ddks(P, Q)
for fl in (0, K.DDKS_FLAG_FORCE_X0, K.DDKS_FLAG_FORCE_DIRECT, K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_TIES_GT,
           K.DDKS_FLAG_RDKS_FULL_SORT | K.DDKS_FLAG_PERM_GATHER):
    with K.Context(flags=fl) as c:
        r = c.stat(dev(P), dev(Q))
        if not fl & K.DDKS_FLAG_TIES_GT:
            assert (r.num, r.argmax_origin) == (want[0], want[3]), (fl, r, want)
        Pb, Qb = I.random_pair(4, 5 * 90, 5 * 70, 5, "grid")
        got = c.stat_batch(dev(Pb.reshape(5, 90, 5)), dev(Qb.reshape(5, 70, 5)))
        assert np.array_equal(got.num, O.batch(Pb.reshape(5, 90, 5), Qb.reshape(5, 70, 5)))
        pooled = np.concatenate([P, Q])
        rng = np.random.default_rng(1)
        perms = np.stack([rng.permutation(len(pooled)) for _ in range(5)]).astype(np.int32)
        null, obs, p = c.permutation_null(dev(pooled), len(P), dev(perms))
        assert np.array_equal(null, O.permutation_null(pooled, len(P), perms)[0])
        s = c.significance(dev(P[:60]), dev(Q[:50]))
        assert s.stat.num == O.ddks(P[:60], Q[:50])[0]
        assert c.vdks(dev(P), dev(Q), 6)[:2] == O.vdks(P, Q, 6)[:2]
        rd = c.rdks(dev(P), dev(Q))
        assert (rd.num, rd.argmax_origin) == (O.rdks(P, Q)[0], O.rdks(P, Q)[3])
torch.cuda.synchronize()
print("sanitize_run ok")
