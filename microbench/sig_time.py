"""Time ddks_significance vs ddks_stat on a BASELINE config (device-resident inputs, CUDA events)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
P, Q = I.config(name)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
    for fn, lab in [(lambda: c.stat(dP, dQ), "stat"), (lambda: c.significance(dP, dQ), "significance"),
                    (lambda: c.significance(dP, dQ, poisson=True), "significance-poisson")]:
        r = fn(); c.profile_read()
        reps = 2 if name == "C5" else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): r = fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        kms, kl, _ = c.profile_read()
        print(f"{name} {lab}: {ms:.3f} ms/call (count kernel {kms / max(kl, 1):.3f} ms) -> {r}", flush=True)
