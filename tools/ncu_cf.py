"""One batched CF split of every level (C2, or CF_CONFIG) inside a
cudaProfilerStart/Stop window, for ncu --profile-from-start off."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

ctx = airg.Context(0)
cfg = int(os.environ.get("CF_CONFIG", "2"))
p = problems.make(cfg)
prm = problems.setup_params(cfg)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
mats = [h.matrix_handle(l, 0) for l in range(h.n_levels)]
seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(h.n_levels)]
labs = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]
airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
for l in range(h.n_levels):
    assert np.array_equal(labs[l][: mats[l].dims()[0]].cpu().numpy(), h.labels(l)), l
print("cf ok", h.n_levels)
