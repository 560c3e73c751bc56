#!/bin/bash
mkdir -p gpurun_out
for V in "" "-DDDKS_C8R=2 -DDDKS_C8T=192" "-DDDKS_C8R=1 -DDDKS_C8T=256"; do
  DDKS_NVCC_EXTRA="$V" python paper_2106_13706_b200/build.py --force > /dev/null 2>&1 || { echo "build failed [$V]"; continue; }
  echo "== variant [$V]"
  python microbench/quick_time.py C3 10 2>&1 | head -1
  DDKS_NO_SMALL=1 python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2106_13706_b200 import ddks as K, inputs as I
P,Q=I.config('C3'); dP,dQ=torch.from_numpy(P).cuda(),torch.from_numpy(Q).cuda()
with K.Context(flags=K.DDKS_FLAG_NO_X0|K.DDKS_FLAG_PROFILE) as c:
    for _ in range(3): c.stat(dP,dQ)
    c.profile_read()
    for _ in range(5): c.stat(dP,dQ)
    ms,n,p=c.profile_read(); print('position-ordered count %.4f ms' % (ms/n))
"
done
