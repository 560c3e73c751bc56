"""ddks_significance_batch vs a loop of ddks_significance on the paper's power-analysis shape (many 50 + 50 tests in
3-D): device-resident inputs, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2106_13706_b200 import ddks as K
rng = np.random.default_rng(5)
B = 4096
Pb = torch.from_numpy(rng.random((B, 50, 3)).astype(np.float32)).cuda()
Qb = torch.from_numpy(rng.random((B, 50, 3)).astype(np.float32)).cuda()
with K.Context() as c:
    c.significance_batch(Pb, Qb)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): r = c.significance_batch(Pb, Qb)
    e1.record(); torch.cuda.synchronize()
    tb = e0.elapsed_time(e1) / 5
    torch.cuda.synchronize(); e0.record()
    for b in range(256): c.significance(Pb[b], Qb[b])
    e1.record(); torch.cuda.synchronize()
    tl = e0.elapsed_time(e1) / 256 * B
    print(f"{B} significance tests (50+50, d=3): batch {tb:.2f} ms, per-pair loop {tl:.1f} ms (extrapolated from 256)")
