"""Batched CF split of all levels of C<argv[1]> (default C2) (the bench's cf_split_ms): median of 10
event-timed airg_cf_split_batch calls; labels checked against the setup's."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

ctx = airg.Context(0)
CFG = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = problems.make(CFG)
prm = problems.setup_params(CFG)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
mats = [h.matrix_handle(l, 0) for l in range(h.n_levels)]
seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(h.n_levels)]
labs = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]
ts = []
for _ in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
    e1.record(ctx.stream)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ok = all(np.array_equal(labs[l][: mats[l].dims()[0]].cpu().numpy(), h.labels(l)) for l in range(h.n_levels))
print(f"C{CFG} cf_split_batch ms median {np.median(ts[2:]):.4f} min {np.min(ts[2:]):.4f} labels_ok {ok}")
