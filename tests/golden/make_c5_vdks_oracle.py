"""Write tests/golden/c5_vdks16_oracle.json: the CPU oracle's vdKS (Alg. 1, literal SumOrthants
over every voxel for every filled voxel) on BASELINE config C5 at k = 16 voxels per dimension -- the configuration
bench.py --method vdks times. About 7 minutes on 8 host threads. Calls only oracle/ and the seeded input generator.
The GPU parity test (tests/test_approx_gpu.py::test_vdks_c5_k16_vs_stored_oracle) compares the kernel's result to it."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

K_VOX = 16
P, Q = I.config("C5")
src = open(os.path.join(ROOT, "oracle", "ddks_oracle.c"), "rb").read()
t0 = time.time()
num, den, D = O.vdks(P, Q, K_VOX)
dt = time.time() - t0
out = {"_source": "tests/golden/make_c5_vdks_oracle.py: oracle.vdks (oracle/ddks_oracle.c, Alg. 1 step by step) on the "
                  "full C5 input, k = 16 (DESIGN.md R15, R16)",
       "config": "C5", "k": K_VOX, "input_sha256": I.sha256_pq(P, Q),
       "oracle_c_sha256": hashlib.sha256(src).hexdigest(),
       "num": num, "den": den, "D_hex": float.hex(D), "seconds": round(dt, 1), "threads": os.cpu_count()}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c5_vdks16_oracle.json"), "w"), indent=1)
print(out)
