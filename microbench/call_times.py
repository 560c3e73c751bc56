"""Wall time of consecutive identical ddks_stat calls: 1st (uncaptured, allocates), 2nd (CUDA-graph capture + launch),
3rd.. (graph replay)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
spec = sys.argv[1] if len(sys.argv) > 1 else "C5"
if ":" in spec:
    d, n = (int(v) for v in spec.split(":"))
    P, Q = I.random_pair(5, n, n, d, "normal")
else:
    P, Q = I.config(spec)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
for fl, lab in [(0, "graph"), (K.DDKS_FLAG_NO_GRAPH, "no-graph")]:
    with K.Context(flags=fl) as c:
        ts = []
        for _ in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter(); c.stat(dP, dQ); ts.append(time.perf_counter() - t0)
        print(spec, lab, " ".join(f"{1e3 * t:.2f}" for t in ts), "ms", flush=True)
