"""Write tests/golden/c5_oracle.json: the CPU oracle's full exact-ddKS statistic on BASELINE config C5 (4*10^12 pair
classifications; hours on a workstation). Calls only oracle/ and the seeded input generator. The GPU parity test
(tests/test_parity_gpu.py::test_config_c5_full_vs_stored_oracle) compares the kernel's whole-C5 result to it."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

P, Q = I.config("C5")
src = open(os.path.join(ROOT, "oracle", "ddks_oracle.c"), "rb").read()
t0 = time.time()
num, den, D, arg = O.ddks(P, Q, threads=os.cpu_count() or 1)
dt = time.time() - t0
out = {"_source": "tests/golden/make_c5_oracle.py: oracle.ddks (oracle/ddks_oracle.c, the paper's loop method) on the "
                  "full C5 input; convention >= (DESIGN.md R1)",
       "config": "C5", "input_sha256": I.sha256_pq(P, Q), "oracle_c_sha256": hashlib.sha256(src).hexdigest(),
       "num": num, "den": den, "D_hex": float.hex(D), "argmax_origin": arg,
       "seconds": round(dt, 1), "threads": os.cpu_count()}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c5_oracle.json"), "w"), indent=1)
print(out)
