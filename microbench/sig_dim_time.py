"""Time ddks_significance for random normal pairs at d = 6..8 (device-resident, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
with K.Context() as c:
    for d in (6, 7, 8):
        P, Q = I.random_pair(d, n, n, d, "normal")
        dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
        r = c.significance(dP, dQ)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(5): r = c.significance(dP, dQ)
        e1.record(); torch.cuda.synchronize()
        print(f"sig d={d} N={2*n}: {e0.elapsed_time(e1)/5:.3f} ms, S={r.S:.4g}", flush=True)
