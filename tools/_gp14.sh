for c in 4 2; do AIRG_SETUP_TIMING=1 python -c "
import sys; sys.path.insert(0,'.')
import time, torch
from paper_2408_08262_b200 import airg, problems
c=$c
p=problems.make(c); prm=dict(problems.setup_params(c), fused_smooths=2)
ctx=airg.Context(0)
dA=airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n,p.n,p.row_offsets,p.cols,p.vals),ctx)
for k in range(2):
    t=time.time(); h=airg.setup(dA, ctx=ctx, **prm); torch.cuda.synchronize(); print('C%d setup %.1f ms'%(c,1e3*(time.time()-t)))
"; done
