cp paper_2106_13706_b200/libddks.so /tmp/o.so
for v in d4 d8 d16; do
  cp variants/rbk_$v.so paper_2106_13706_b200/libddks.so; echo "== $v"
  timeout 200 python microbench/graph_ab.py 30 2>&1 | grep rdks
  timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np
from paper_2106_13706_b200 import ddks as K, inputs as I
for c in ['C2','C3']:
    P,Q=I.config(c); dP,dQ=torch.from_numpy(P).cuda(),torch.from_numpy(Q).cuda()
    with K.Context() as x:
        for _ in range(4): x.rdks(dP,dQ)
        torch.cuda.synchronize(); e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record()
        for _ in range(30): r=x.rdks(dP,dQ)
        e1.record(); torch.cuda.synchronize(); print(c, 'rdks %.1f us' % (e0.elapsed_time(e1)/30*1e3))
"
done
cp /tmp/o.so paper_2106_13706_b200/libddks.so
