"""One-GPU rehearsal of the multi-GPU C5 statistic: for world = 1, 2, 4, 8, time on this device the
origin shard every rank would own (ddks_stat_shard: the same kernels, shard of the kd order, no collective),
combine the shard results as NCCL would, and report the projected per-world time = max over ranks. This is a
projection from one B200, not a multi-GPU measurement (the NCCL all-reduce of one uint64 is not included)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
P, Q = I.config(name)
dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
out = {"workload": name, "note": __doc__.split("\n\n")[0].replace("\n", " "), "worlds": {}}
with K.Context() as c:
    c.stat(dP, dQ)  # warm-up
    for world in (1, 2, 4, 8):
        times, parts = [], []
        for r in range(world):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            parts.append(c.stat_shard(dP, dQ, world, r))
            e1.record(); torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        num = max(p.num for p in parts)
        arg = min(p.argmax_origin for p in parts if p.num == num)
        out["worlds"][world] = {"rank_ms": [round(t, 3) for t in times], "projected_ms": round(max(times), 3),
                                "num": num, "argmax_origin": arg}
        print(world, out["worlds"][world], flush=True)
t1 = out["worlds"][1]["projected_ms"]
for w, v in out["worlds"].items():
    v["projected_efficiency"] = round(t1 / (w * v["projected_ms"]), 4)
print(json.dumps(out))
