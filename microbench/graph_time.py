"""ddks_stat per-call wall time and device time, CUDA graph replay vs uncaptured (DDKS_FLAG_NO_GRAPH), small configs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
for name in sys.argv[1:] or ["C1", "C2"]:
    P, Q = I.config(name)
    dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    for lab, fl in [("graph", 0), ("no-graph", K.DDKS_FLAG_NO_GRAPH)]:
        with K.Context(flags=fl) as c:
            for _ in range(5): c.stat(dP, dQ)
            n = 300
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record()
            for _ in range(n): c.stat(dP, dQ)
            e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
            print(f"{name} {lab:9s} wall {1e3 * (t1 - t0) / n:.4f} ms/call  device {e0.elapsed_time(e1) / n:.4f} ms/call",
                  flush=True)
