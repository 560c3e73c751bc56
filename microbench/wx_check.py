import sys, os
sys.path.insert(0, '.')
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
P, Q = I.config('C2'); dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
for env in [None, "1"]:
    if env: os.environ["DDKS_NO_WX"] = env
    with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
        for _ in range(3): c.stat(dP, dQ)
        c.profile_read(); c.profile_work()
        for _ in range(10): r = c.stat(dP, dQ)
        ms, n, pairs = c.profile_read(); ex = c.profile_work()
        print("NO_WX" if env else "WX", "count ms %.4f" % (ms / n), "launches/call", n / 10, "compares/pair %.3f" % (ex / pairs), r)
