"""One C3 ddks_stat through the rank-lane count (forced, so C2 takes it too), for ncu captures (dev helper)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2106_13706_b200 import ddks as K, inputs as I
P, Q = I.config(sys.argv[1] if len(sys.argv) > 1 else "C3")
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
with K.Context(flags=K.DDKS_FLAG_NO_GRAPH | K.DDKS_FLAG_FORCE_RANK) as c:
    for _ in range(2):
        r = c.stat(dP, dQ)
    torch.cuda.synchronize()
    print(r)
