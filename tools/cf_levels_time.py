"""Per-level CF split time (fused split, C2) under the current AIRG_CF_* env:
median of 5 event-timed calls per level. Usage: python tools/cf_levels_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

CFG = int(os.environ.get("CF_CONFIG", "2"))
p = problems.make(CFG)
prm = problems.setup_params(CFG)
ctx = airg.default_context()
h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx=ctx, **prm)
stream = ctx.stream
tot = 0.0
only = os.environ.get("CF_LEVELS")
for l in range(h.n_levels):
    if only is not None and str(l) not in only.split(","):
        continue
    A = h.matrix_handle(l, 0)
    n = A.dims()[0]
    seed = int(problems.mix(np.uint64(0), np.uint64(l)))
    lab = ctx.empty(max(n, 1), torch.uint8)
    ts = []
    for _ in range(int(os.environ.get("CF_REPS", "6"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        airg.cf_split_batch_device([A], [seed], prm["strength_alpha"], prm["max_loops"], labels=[lab], ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    med = float(np.median(ts[1:] if len(ts) > 1 else ts))
    tot += med
    print(f"{l:3d} {n:9d} {h.level(l).nnz:10d} {h.level(l).nnz / max(n, 1):6.1f} {med:8.1f}")
print(f"total {tot:.1f} us")
