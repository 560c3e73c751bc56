"""C4 step split into its two C-ABI calls (batch statistic, permutation null), each device-timed with CUDA events
around the call, with and without DDKS_FLAG_PROFILE; plus the raw C-ABI call cost of each."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I

P, Q = I.config("C4")
perms = I.c4_perms()
pooled = np.concatenate([P[I.C4_PERM_PAIR], Q[I.C4_PERM_PAIR]])
n = P.shape[1]
dP, dQ, dpool, dperm = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P, Q, pooled, perms))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.median(ts) * 1e3


for lab, fl in [("plain", 0), ("profile", K.DDKS_FLAG_PROFILE)]:
    with K.Context(flags=fl) as c:
        tb = timed(lambda: c.stat_batch(dP, dQ))
        tn = timed(lambda: c.permutation_null(dpool, n, dperm))
        tboth = timed(lambda: (c.stat_batch(dP, dQ), c.permutation_null(dpool, n, dperm)))
        print(f"{lab:8s} stat_batch {tb:8.1f} us   permutation_null {tn:8.1f} us   both {tboth:8.1f} us", flush=True)
