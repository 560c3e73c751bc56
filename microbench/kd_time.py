"""kd ordering: time ddks_stat (whole call and count kernel, CUDA events / DDKS_FLAG_PROFILE) per DDKS_KD setting.
usage: kd_time.py <config | d:n> <reps> <setting> ...   setting = "auto" | "K" | "K,G0,G1"; d:n = random normal
pair of n + n points in d dims."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
name, reps = sys.argv[1], int(sys.argv[2])
if ":" in name:
    d, n = (int(v) for v in name.split(":"))
    P, Q = I.random_pair(5, n, n, d, "normal")
else:
    P, Q = I.config(name)
d = P.shape[1]
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
ref = None
for setting in sys.argv[3:]:
    if setting == "auto":
        os.environ.pop("DDKS_KD", None)
    else:
        os.environ["DDKS_KD"] = setting
    with K.Context(flags=K.DDKS_FLAG_PROFILE | K.DDKS_FLAG_FORCE_X0) as c:
        r = c.stat(dP, dQ)
        c.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): r = c.stat(dP, dQ)
        e1.record(); torch.cuda.synchronize()
        kms, nl, pairs = c.profile_read()
        ms = e0.elapsed_time(e1) / reps
        frac = d * pairs / (kms / 1e3) / 18.61e12
        ref = ref or r
        print(f"{name} kd={setting:10s} levels={c.kd_levels} call {ms:9.3f} ms  count {kms / nl:9.3f} ms  "
              f"compare-roofline frac {frac:.3f}  same={r == ref}", flush=True)
