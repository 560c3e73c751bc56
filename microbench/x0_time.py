"""Time ddks_stat on a config with the x0-ordered kernel forced on vs off (device-resident inputs, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
for name in sys.argv[1:]:
    P, Q = I.config(name)
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    for lab, fl in [("x0", K.DDKS_FLAG_FORCE_X0), ("no-x0", K.DDKS_FLAG_NO_X0)]:
        with K.Context(flags=fl) as c:
            r = c.stat(dP, dQ)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): r = c.stat(dP, dQ)
            e1.record(); torch.cuda.synchronize()
            print(name, lab, round(e0.elapsed_time(e1) / 20, 4), "ms", r, flush=True)
