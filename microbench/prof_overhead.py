"""Per-call device time with and without DDKS_FLAG_PROFILE (dev helper): the cost of the in-kernel probes."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2106_13706_b200 import ddks as K, inputs as I
reps = 50
for name in sys.argv[1:] or ["C1", "C2", "C3"]:
    P, Q = I.config(name)
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    out = {}
    for flags, tag in ((0, "plain"), (K.DDKS_FLAG_PROFILE, "profile")):
        c = K.Context(flags=flags)
        f = (lambda: c.stat_batch(dP, dQ)) if name == "C4" else (lambda: c.stat(dP, dQ))
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f()
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
        out[tag] = min(ts)
    print(name, "ms/call plain %.4f profile %.4f (+%.1f us)" % (out["plain"], out["profile"], 1e3 * (out["profile"] - out["plain"])))
