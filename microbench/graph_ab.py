"""Per-call device time of each C-ABI call with and without its CUDA graph (DDKS_FLAG_NO_GRAPH): back-to-back calls,
CUDA events around reps calls (each call syncs inside). argv: reps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
P5, Q5 = I.config("C5")
P2, Q2 = I.config("C2")
P3, Q3 = I.config("C3")
P4, Q4 = I.config("C4")
perms = I.c4_perms()
pooled = np.concatenate([P4[I.C4_PERM_PAIR], Q4[I.C4_PERM_PAIR]])
d5 = [torch.from_numpy(a).cuda() for a in (P5, Q5)]
d2 = [torch.from_numpy(a).cuda() for a in (P2, Q2)]
d3 = [torch.from_numpy(a).cuda() for a in (P3, Q3)]
d4 = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P4, Q4, pooled, perms)]
calls = {
    "vdks C5 k16": lambda c: c.vdks(d5[0], d5[1], 16),
    "rdks C5": lambda c: c.rdks(d5[0], d5[1]),
    "stat C2": lambda c: c.stat(d2[0], d2[1]),
    "stat C3": lambda c: c.stat(d3[0], d3[1]),
    "batch C4": lambda c: c.stat_batch(d4[0], d4[1]),
    "null C4": lambda c: c.permutation_null(d4[2], 512, d4[3]),
}
for name, f in calls.items():
    out = []
    for fl in (0, K.DDKS_FLAG_NO_GRAPH):
        with K.Context(flags=fl) as c:
            for _ in range(4):
                f(c)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f(c)
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) / reps * 1e3)
    print(f"{name:14s} graph {out[0]:9.1f} us   no graph {out[1]:9.1f} us", flush=True)
