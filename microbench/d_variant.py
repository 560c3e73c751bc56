"""Time ddks_stat for one d at N = 2n (random normal, x0 forced) for each given library build (A/B of geometries)."""
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2106_13706_b200", "libddks.so")
code = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2106_13706_b200 import ddks as K, inputs as I
d, n = int(sys.argv[1]), int(sys.argv[2])
P, Q = I.random_pair(d, n, n, d, "normal")
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context(flags=K.DDKS_FLAG_FORCE_X0) as c:
    r = c.stat(dP, dQ)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): r = c.stat(dP, dQ)
    e1.record(); torch.cuda.synchronize()
    print(round(e0.elapsed_time(e1) / 5, 3), r.num)
''' % ROOT
d, n = sys.argv[1], sys.argv[2]
for so in sys.argv[3:]:
    shutil.copy(so, SO)
    out = subprocess.run([sys.executable, "-c", code, d, n], capture_output=True, text=True)
    print(os.path.basename(so), out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
