"""A/B timing of library builds: for each .so given, copy it in place and time ddks_stat on a config in a fresh
process (device-resident inputs, CUDA events)."""
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2106_13706_b200", "libddks.so")
code = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2106_13706_b200 import ddks as K, inputs as I
P, Q = I.config(sys.argv[1]); n = int(sys.argv[2])
if n: P, Q = P[:n].copy(), Q[:n].copy()
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context(flags=int(sys.argv[3])) as c:
    r = c.stat(dP, dQ)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): r = c.stat(dP, dQ)
    e1.record(); torch.cuda.synchronize()
    print(round(e0.elapsed_time(e1) / 5, 3), r.num)
''' % ROOT
# usage: variant_time.py CONFIG N_PER_SAMPLE(0 = all) FLAGS lib1.so lib2.so ...
cfg, n, flags = sys.argv[1:4]
for so in sys.argv[4:]:
    shutil.copy(so, SO)
    out = subprocess.run([sys.executable, "-c", code, cfg, n, flags], capture_output=True, text=True)
    print(os.path.basename(so), out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
