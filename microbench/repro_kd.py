import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from oracle import oracle as O
from paper_2106_13706_b200 import ddks as K, inputs as I
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
bad = 0
for (nP, nQ) in [(31, 512), (512, 31), (300, 200), (33, 4097), (2000, 1500)]:
    for d in range(2, 9):
        for kind in ["normal", "grid", "mixed", "dup"]:
            P, Q = I.random_pair(11 + d, nP, nQ, d, kind)
            w = O.ddks(P, Q)
            for fl, lab in [(K.DDKS_FLAG_FORCE_X0, "x0"), (K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_FORCE_DIRECT, "x0direct")]:
                with K.Context(flags=fl) as c:
                    r = c.stat(dev(P), dev(Q))
                    if (r.num, r.argmax_origin) != (w[0], w[3]):
                        bad += 1
                        if bad < 15: print("MISMATCH", lab, nP, nQ, d, kind, (r.num, r.argmax_origin), (w[0], w[3]), "K", c.kd_levels)
print("bad", bad)
