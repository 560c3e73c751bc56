"""vdKS (k=16) / rdKS at C5: per-call device time (CUDA events); argv[1] = reps (dev helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
which = sys.argv[2:] or ["vdks", "rdks"]
P, Q = I.config("C5")
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context() as c:
    for m in which:
        f = (lambda: c.vdks(dP, dQ, 16)) if m == "vdks" else (lambda: c.rdks(dP, dQ))
        r = f(); r = f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r = f()
        e1.record(); torch.cuda.synchronize()
        print(f"C5 {m}: {e0.elapsed_time(e1) / reps:.4f} ms/call -> {r}", flush=True)
