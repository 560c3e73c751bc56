"""Seeded fuzz of the mid-N kd path (cluster ordering; FORCE_X0 so every d takes it) against the oracle at N between
20 000 and 70 000 -- label runs from a few hundred rows to past one cluster slice, every d, tie-heavy kinds -- plus
the same inputs through the fused cooperative ordering (DDKS_KD_FUSED). argv: cases (default 16)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2106_13706_b200 import ddks as K, inputs as I

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(77)
bad = 0
with K.Context(flags=K.DDKS_FLAG_FORCE_X0) as c:
    for i in range(n_cases):
        N = int(rng.integers(20000, 70001))
        n_P = int(rng.integers(300, N - 300))
        d = int(rng.integers(2, 9))
        kind = str(rng.choice(["normal", "grid", "mixed", "dup"]))
        P, Q = I.random_pair(int(rng.integers(0, 2**31)), n_P, N - n_P, d, kind)
        t0 = time.time()
        want = O.ddks(P, Q)
        t_or = time.time() - t0
        dP, dQ = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
        os.environ.pop("DDKS_KD_FUSED", None)
        r = c.stat(dP, dQ)
        lv = c.kd_levels
        os.environ["DDKS_KD_FUSED"] = "1"
        rf = c.stat(dP, dQ)
        os.environ.pop("DDKS_KD_FUSED", None)
        ok = (r.num, r.den, r.argmax_origin) == (want[0], want[1], want[3]) and rf == r
        bad += not ok
        print(f"case {i:2d} N={N} n_P={n_P} d={d} {kind:6s} kd_levels={lv} num={r.num} oracle={want[0]} "
              f"argmax {r.argmax_origin}/{want[3]} fused_same={rf == r} {'OK' if ok else 'MISMATCH'} ({t_or:.1f} s oracle)",
              flush=True)
print(f"{n_cases - bad}/{n_cases} cases bit-exact")
sys.exit(1 if bad else 0)
