"""rdKS at the paper's high-dimensional shape (100 points per sample in 1000 dimensions, "approximately 4 s"):
device-resident inputs, CUDA events; checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2106_13706_b200 import ddks as K
rng = np.random.default_rng(11)
d = 1000
P = rng.random((100, d)).astype(np.float32)                       # "uniform" sample
u = rng.random((100, 1))
Q = np.clip(u + 0.05 * rng.standard_normal((100, d)), 0, 1).astype(np.float32)  # "diagonal" sample
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context() as c:
    r = c.rdks(dP, dQ)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): r = c.rdks(dP, dQ)
    e1.record(); torch.cuda.synchronize()
    o = O.rdks(P, Q)
    assert (r.num, r.argmax_origin) == (o[0], o[3])
    print(f"rdKS n=100+100 d=1000: {e0.elapsed_time(e1) / 20:.3f} ms per statistic on the device, D={r.D}, corner {r.argmax_origin} (oracle agrees)")
