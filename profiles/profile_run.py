"""Short run of the production kernels for ncu captures (ncu replays every kernel ~500x with --set full, so the
full C5 statistic (1.4 s per launch) is too long to profile; this runs the SAME k_count instantiation and launch
configuration on an origin subset via ddks_stat_per_origin, or a whole small config).

    python profiles/profile_run.py C5 <o_begin> <o_end>   # C5 origin subset (same kernel, same segments)
    python profiles/profile_run.py C3|C2|C1               # full statistic
    python profiles/profile_run.py C4                     # full 4096-pair batch
    python profiles/profile_run.py C5kd <n>               # first n + n points of C5 through the kd-ordered kernel
                                                          # (same k_count<5, ., ., K> kernel and CTA shape; the cost
                                                          # model picks the cuts for n, so K / cells differ from C5)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

name = sys.argv[1]
flags = 0
if name in ("C5x0", "C5kd"):
    P, Q = I.config("C5")
    n = int(sys.argv[2])
    P, Q = P[:n].copy(), Q[:n].copy()
    flags = K.DDKS_FLAG_FORCE_X0
    sys.argv = sys.argv[:2]
else:
    P, Q = I.config(name)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context(flags=flags | K.DDKS_FLAG_PROFILE) as c:
    for i in range(2):
        if name == "C4":
            r = c.stat_batch(dP, dQ)[0]
        elif len(sys.argv) > 3:
            r = int(c.stat_per_origin(dP, dQ, int(sys.argv[2]), int(sys.argv[3])).max())
        else:
            r = c.stat(dP, dQ)
        # executed FP32 compares of this call's count kernel(s) (in-kernel counter; ncu's FSET count x 32 must match)
        print(name, "call", i, "executed_compares", c.profile_work(), "kd_levels", c.kd_levels, flush=True)
    torch.cuda.synchronize()
    print(name, r, "launches", c.launch_count)
