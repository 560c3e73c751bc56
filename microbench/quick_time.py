"""Quick device timing of ddks_stat on a config (dev helper; bench.py is the contract)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2106_13706_b200 import ddks as K, inputs as I
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P, Q = I.config(name)
if name == "C4":
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
else:
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
c = K.Context(flags=K.DDKS_FLAG_PROFILE)
f = (lambda: c.stat_batch(dP, dQ)) if name == "C4" else (lambda: c.stat(dP, dQ))
r = f()
torch.cuda.synchronize()
c.profile_read()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = f(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
N = (P.shape[-2] + Q.shape[-2])
pairs = N * N * (P.shape[0] if name == "C4" else 1)
kms, kl, kp = c.profile_read()
ms = min(ts)
print("kernel-only: %.4f ms/launch, %.3e pairs/s, frac %.3f" % (kms / kl, kp / kms * 1e3, kp / kms * 1e3 * P.shape[-1] / (148 * 64 * 1.965e9)))
d = P.shape[-1]
print(name, "ms", ts, "pairs/s %.3e" % (pairs / ms * 1e3), "frac_alu(1965MHz) %.3f" % (pairs / ms * 1e3 * d / (148 * 64 * 1.965e9)),
      (r[0] if name == "C4" else r))
