"""Setup wall time (median of 3, after one warm-up) of a config, with the
fast V-cycle's fused operators built as the bench does (fused_smooths = 2).
  [AIRG_SETUP_TIMING=1] python tools/setup_probe.py [--config 4]"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--fused", type=int, default=2)
a = ap.parse_args()
ctx = airg.Context(0)
p = problems.make(a.config)
prm = dict(problems.setup_params(a.config), fused_smooths=a.fused)
dA = airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx)
ts = []
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = airg.setup(dA, ctx=ctx, **prm)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
    if k < 3:
        del h
ts = sorted(ts[1:])
print(f"C{a.config} setup ms: median {ts[1]:.1f} (min {ts[0]:.1f}), levels {h.n_levels}, plan {h.fused_plan()}")
