"""Sweep the forced point-segment count (DDKS_SEGS) for one config's statistic; prints kernel ms per segs."""
import os, subprocess, sys
name = sys.argv[1]
for segs in sys.argv[2:]:
    env = dict(os.environ, DDKS_SEGS=segs)
    out = subprocess.run([sys.executable, "bench.py", "--workload", name, "--steps", "5", "--warmup", "3",
                          "--no-cpu-baseline", "--no-e2e"], env=env, capture_output=True, text=True).stdout
    import json
    d = json.loads(out.strip().splitlines()[-1])
    print(name, "segs", segs, "step ms", round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 4), flush=True)
