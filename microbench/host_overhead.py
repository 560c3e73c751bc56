"""Per-call cost of a small statistic (C1) split into its parts: the floor of a torch launch + sync, the raw C-ABI
call with prebuilt ctypes arguments (CUDA-graph replay), and the Python binding around it."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


name = sys.argv[1] if len(sys.argv) > 1 else "C1"
P, Q = I.config(name)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
x = torch.zeros(1, device="cuda")
print(f"torch add_ + synchronize        {per_call(lambda: (x.add_(1), torch.cuda.synchronize())):8.2f} us")
print(f"torch synchronize alone         {per_call(torch.cuda.synchronize):8.2f} us")
for lab, fl in [("graph", 0), ("no-graph", K.DDKS_FLAG_NO_GRAPH), ("graph+profile", K.DDKS_FLAG_PROFILE)]:
    with K.Context(flags=fl) as c:
        r = K.ddks_result()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        args = (c.ctx, ctypes.c_void_p(dP.data_ptr()), P.shape[0], ctypes.c_void_p(dQ.data_ptr()), Q.shape[0], P.shape[1],
                st, ctypes.byref(r))
        raw = per_call(lambda: K.LIB.ddks_stat(*args))
        py = per_call(lambda: c.stat(dP, dQ))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(20):
            c.stat(dP, dQ)
        e0.record()
        for _ in range(500):
            c.stat(dP, dQ)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {lab:14s} raw C-ABI {raw:8.2f} us   python binding {py:8.2f} us   device-timed "
              f"{e0.elapsed_time(e1) / 500 * 1e3:8.2f} us/call", flush=True)
