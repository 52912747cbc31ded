"""Per-Richardson-iteration cost on C2 from solves capped at k iterations
(device loop and host loop), to expose per-iteration launch overhead."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

ctx = airg.Context(0)
p = problems.make(2)
prm = problems.setup_params(2)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
tb = ctx.to_device(p.b)
tx = ctx.empty(p.n, torch.float64)
res = {}
for k in (2, 4, 8, 16):
    sk = dict(coarse_iterations=3, max_iterations=k, rtol=1e-30)
    h.solve_device(tb, tx, **sk)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        st, _ = h.solve_device(tb, tx, **sk)
        e1.record(ctx.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[k] = float(np.median(ts))
print("devloop" if os.environ.get("AIRG_DEVLOOP", "1") != "0" else "hostloop",
      {k: round(v, 3) for k, v in res.items()}, "per-iteration ms:", round((res[16] - res[8]) / 8, 4))
