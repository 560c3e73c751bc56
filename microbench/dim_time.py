"""Time ddks_stat for random normal pairs at each d (device-resident, CUDA events): kernel-design sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
x0 = len(sys.argv) > 2 and sys.argv[2] == "x0"
with K.Context(flags=K.DDKS_FLAG_PROFILE | (K.DDKS_FLAG_FORCE_X0 if x0 else K.DDKS_FLAG_NO_X0)) as c:
    for d in range(1, 9):
        P, Q = I.random_pair(d, n, n, d, "normal")
        dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
        r = c.stat(dP, dQ); c.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): r = c.stat(dP, dQ)
        e1.record(); torch.cuda.synchronize()
        ms, nl, pairs = c.profile_read()
        frac = d * pairs / (ms / 1e3) / (148 * 64 * 1.965e9)
        print(f"{'x0' if x0 else 'pos'} d={d} N={2*n} step {e0.elapsed_time(e1)/10:.3f} ms kernel {ms/nl:.3f} ms frac {frac:.3f}", flush=True)
