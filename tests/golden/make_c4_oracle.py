"""Write tests/golden/c4_oracle.json: the CPU oracle's num for EVERY item of BASELINE config C4a (4096 independent
pairs, d = 4, 512 + 512) and EVERY permutation of C4b (1000 label shuffles of pair 2048), plus the observed num and
the add-one p-value. Calls only oracle/ and the seeded input generator (seconds on a few host threads).
The GPU parity test (tests/test_parity_gpu.py::test_config_c4_every_item_and_permutation) compares the kernels'
results element by element to this file and to a live oracle run; tests/test_oracle_pins.py pins the file to the
survey's independently computed aggregates."""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402

P, Q = I.config("C4")
perms = I.c4_perms()
pooled = np.concatenate([P[I.C4_PERM_PAIR], Q[I.C4_PERM_PAIR]])
src = open(os.path.join(ROOT, "oracle", "ddks_oracle.c"), "rb").read()
t0 = time.time()
batch = O.batch(P, Q, threads=os.cpu_count() or 1)
null, obs, p_num, p_val = O.permutation_null(pooled, P.shape[1], perms, threads=os.cpu_count() or 1)
dt = time.time() - t0
out = {"_source": "tests/golden/make_c4_oracle.py: oracle.batch and oracle.permutation_null (oracle/ddks_oracle.c, the "
                  "paper's loop method per item / per permutation) on the full C4 input; convention >= (DESIGN.md R1)",
       "config": "C4", "input_sha256": I.sha256_pq(P, Q),
       "perms_sha256": hashlib.sha256(perms.tobytes()).hexdigest(),
       "oracle_c_sha256": hashlib.sha256(src).hexdigest(),
       "den": int(P.shape[1]) * int(Q.shape[1]),
       "batch_num": [int(v) for v in batch],
       "perm_pair": I.C4_PERM_PAIR, "observed_num": obs, "null_num": [int(v) for v in null],
       "p_num": p_num, "p_value": p_val, "seconds": round(dt, 1), "threads": os.cpu_count()}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c4_oracle.json"), "w"))
print({k: v for k, v in out.items() if k not in ("batch_num", "null_num")})
