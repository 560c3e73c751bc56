"""ddks_stat call time, kd-ordered (DDKS_FLAG_FORCE_X0) vs position-ordered (DDKS_FLAG_NO_X0), for n + n random
normal points: where the kd sort starts to pay (the library's threshold, x0_applicable)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
for d in [int(v) for v in sys.argv[1].split(",")]:
    for n in [int(v) for v in sys.argv[2].split(",")]:
        P, Q = I.random_pair(3, n, n, d, "normal")
        dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
        res = []
        for fl in (K.DDKS_FLAG_FORCE_X0, K.DDKS_FLAG_NO_X0):
            with K.Context(flags=fl) as c:
                for _ in range(3): r = c.stat(dP, dQ)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record()
                for _ in range(10): r2 = c.stat(dP, dQ)
                e1.record(); torch.cuda.synchronize()
                res.append(e0.elapsed_time(e1) / 10)
                assert r2 == r
        print(f"d={d} N={2 * n}: kd {res[0]:.3f} ms, position {res[1]:.3f} ms, ratio {res[1] / res[0]:.2f}", flush=True)
