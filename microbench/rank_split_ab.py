"""SPLIT rank-lane count (two launches over the P and the Q rows) vs the FP32 SPLIT counts: warm call times of
ddks_significance and of ddks_stat at sample sizes that need SPLIT counters. Usage: python microbench/rank_split_ab.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2106_13706_b200 import ddks as K, inputs as I


def timed(f, reps=7):
    f(); f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return r, float(np.median(ts))


modes = [("rank", K.DDKS_FLAG_FORCE_RANK), ("fp32-auto", K.DDKS_FLAG_NO_RANK), ("fp32-pos", K.DDKS_FLAG_NO_RANK | K.DDKS_FLAG_NO_X0)]
NS = (10000, 20000, 40000, 100000, 200000)
for a in sys.argv[1:]:
    if a.startswith("--n="):
        NS = tuple(int(x) for x in a[4:].split(","))
for what in ("significance", "stat"):
    for d in (8, 7, 6, 5, 3):
        for n in NS:
            # stat: n_P = n/2 + 1, n_Q = n/2 (coprime: SPLIT counters); significance: equal sizes
            n_P, n_Q = (n // 2, n // 2) if what == "significance" else (n // 2 + 1, n // 2)
            P, Q = I.random_pair(5151 + n + d, n_P, n_Q, d, "normal")
            dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
            line, res = f"{what} d{d} N{n}", {}
            for mname, fl in modes:
                with K.Context(flags=fl) as c:
                    f = (lambda: c.significance(dP, dQ)) if what == "significance" else (lambda: c.stat(dP, dQ))
                    r, ms = timed(f, reps=3 if n >= 100000 else 7)
                    res[mname] = (r.stat.num, r.stat.argmax_origin, r.log_prod) if what == "significance" else (r.num, r.argmax_origin)
                    line += f"  {mname}: {ms:.4f} ms (rank={c.rank_lanes} kd={c.kd_levels})"
            print(line, " same=%s" % (len(set(res.values())) == 1), flush=True)
