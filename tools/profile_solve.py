"""Profiling driver: build the C2 hierarchy, warm up, then run ONE solve
between cudaProfilerStart/Stop so `ncu --profile-from-start off` captures
exactly the kernels of one timed step (setup excluded).

  python tools/profile_solve.py [--config 2] [--what solve|spmv|setup]
"""
import argparse
import os
import sys

import numpy as np

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--what", default="solve")
    ap.add_argument("--outer", type=int, default=None, help="1 = outer GMRES(30) (default for C0 / C4)")
    ap.add_argument("--fast", type=int, default=1, help="1 = fast mode (the bench's), 0 = exact")
    args = ap.parse_args()
    # profilers do not see the kernels of conditional graph bodies: Richardson
    # runs its host-driven loop (AIRG_DEVLOOP=0), GMRES the device-resident
    # kernels launched one by one (AIRG_GM_FLAT=1)
    gm = args.outer if args.outer is not None else int(args.config in (0, 4))
    if gm:
        os.environ.setdefault("AIRG_GM_FLAT", "1")
    else:
        os.environ.setdefault("AIRG_DEVLOOP", "0")
    ctx = airg.Context(0)
    p = problems.make(args.config, args.scale)
    prm = dict(problems.setup_params(args.config), fused_smooths=2 if args.fast else -1)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    if args.what == "setup":
        airg.setup(dA, ctx=ctx, **prm)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        h = airg.setup(dA, ctx=ctx, **prm)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    h = airg.setup(dA, ctx=ctx, **prm)
    tb = ctx.to_device(p.b)
    tx = ctx.empty(p.n, torch.float64)
    outer = args.outer if args.outer is not None else int(args.config in (0, 4))
    sk = dict(coarse_iterations=prm["coarse_iterations"], outer=outer, fast=args.fast, max_iterations=400)
    for _ in range(2):
        st, _ = h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    if args.what == "spmv":
        A0 = h.matrix_handle(0, 0)
        x = torch.rand(p.n, dtype=torch.float64, device=ctx.tdev)
        y = torch.empty_like(x)
        airg.spmv_device(A0, x, y, ctx=ctx)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(3):
            airg.spmv_device(A0, x, y, ctx=ctx)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    torch.cuda.profiler.start()
    st, _ = h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("iterations", st.iterations, "levels", h.n_levels)


if __name__ == "__main__":
    main()
