"""C2 / C3 / C1 count time vs the number of point segments (DDKS_SEGS override) — checks the segment chooser."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
name = sys.argv[1]
P, Q = I.config(name)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
for sg in ["auto"] + sys.argv[2:]:
    if sg == "auto":
        os.environ.pop("DDKS_SEGS", None)
    else:
        os.environ["DDKS_SEGS"] = sg
    with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
        for _ in range(3): c.stat(dP, dQ)
        c.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(50): r = c.stat(dP, dQ)
        e1.record(); torch.cuda.synchronize()
        kms, nl, _ = c.profile_read()
        print(name, "segs", sg, "call", round(e0.elapsed_time(e1) / 50, 4), "count", round(kms / nl, 4), r.num, flush=True)
