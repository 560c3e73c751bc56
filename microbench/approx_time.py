"""Time vdKS (and rdKS when built) on BASELINE configs, device-resident inputs, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
for name, ks in [("C2", [16, 32, 64]), ("C3", [2, 4]), ("C5", [8, 16, 24])]:
    P, Q = I.config(name)
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    with K.Context() as c:
        for k in ks:
            r = c.vdks(dP, dQ, k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): r = c.vdks(dP, dQ, k)
            e1.record(); torch.cuda.synchronize()
            print(f"{name} vdks k={k}: {e0.elapsed_time(e1) / 5:.3f} ms -> {r}", flush=True)
        if hasattr(c, "rdks"):
            r = c.rdks(dP, dQ)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): r = c.rdks(dP, dQ)
            e1.record(); torch.cuda.synchronize()
            print(f"{name} rdks: {e0.elapsed_time(e1) / 5:.3f} ms -> {r}", flush=True)
