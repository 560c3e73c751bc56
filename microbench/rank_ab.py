"""Rank-lane count (ddks_rank.cuh) vs the FP32 counts: warm ddks_stat call time (graphed) and count-kernel time,
results compared. Usage: python microbench/rank_ab.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2106_13706_b200 import ddks as K, inputs as I


def timed(c, f, reps=7):
    f(); f(); torch.cuda.synchronize()
    c.profile_read()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    kms, kl, kp = c.profile_read()
    return r, float(np.median(ts)), kms / max(kl, 1) * 1.0


NS = (10000, 20000, 40000, 100000, 400000)
args = sys.argv[1:]
for a in list(args):  # --n=60000,80000: other sizes (threshold search)
    if a.startswith("--n="):
        NS = tuple(int(x) for x in a[4:].split(","))
        args.remove(a)
cases = [("C3", None), ("C2", None)] + [(f"d{d} N{n}", (d, n)) for d in (8, 7, 6, 5, 4, 3, 2) for n in NS]
if args:
    cases = [c for c in cases if any(s in c[0] for s in args)]
modes = [("rank", K.DDKS_FLAG_FORCE_RANK), ("fp32-auto", K.DDKS_FLAG_NO_RANK), ("fp32-pos", K.DDKS_FLAG_NO_RANK | K.DDKS_FLAG_NO_X0)]
for name, spec in cases:
    if spec is None:
        P, Q = I.config(name)
    else:
        d, n = spec
        P, Q = I.random_pair(4242 + n + d, n // 2, n // 2, d, "normal")
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    res = {}
    line = name
    for mname, fl in modes:
        with K.Context(flags=fl | K.DDKS_FLAG_PROFILE) as c:
            r, ms, kms = timed(c, lambda: c.stat(dP, dQ), reps=3 if P.shape[0] >= 200000 else 7)
            res[mname] = (r.num, r.argmax_origin)
            line += f"  {mname}: call {ms:.4f} ms count {kms:.4f} ms kd={c.kd_levels}"
    same = len(set(res.values())) == 1
    print(line, " same=%s" % same, flush=True)
