"""Per-iteration solve timings of the loop implementations (device-resident
conditional graphs vs the host-driven loops), C4 by default.
  AIRG_DEVLOOP=0|1 python tools/gm_probe.py [--config 4] [--fast 1]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--fast", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--profile", action="store_true",
                    help="one GMRES(30) cycle between cudaProfilerStart/Stop (ncu --profile-from-start off)")
    a = ap.parse_args()
    ctx = airg.Context(0)
    p = problems.make(a.config)
    prm = dict(problems.setup_params(a.config), fused_smooths=2 if a.fast else -1)
    h = airg.setup(airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx),
                   ctx=ctx, **prm)
    if a.fast:
        plan = h.fused_plan()
        print("one-pass levels:", [l for l, v in enumerate(plan["one_pass"]) if v],
              "coarse composed:", plan["coarse_composed"])
    tb = ctx.to_device(p.b)
    tx = ctx.empty(p.n, torch.float64)
    if a.profile:
        kw = dict(outer=1, max_iterations=30, coarse_iterations=prm["coarse_iterations"], fast=a.fast)
        h.solve_device(tb, tx, **kw)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        h.solve_device(tb, tx, **kw)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    for name, kw in (("richardson x8", dict(outer=0, max_iterations=8)),
                     ("gmres x30", dict(outer=1, max_iterations=30)),
                     ("gmres full", dict(outer=1, max_iterations=400))):
        kw = dict(kw, coarse_iterations=prm["coarse_iterations"], fast=a.fast)
        for _ in range(2):
            st, _ = h.solve_device(tb, tx, **kw)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            st, _ = h.solve_device(tb, tx, **kw)
            e1.record(ctx.stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"{name:14s} devloop={os.environ.get('AIRG_DEVLOOP', '1')} fast={a.fast}: {ms:8.3f} ms, "
              f"{st.iterations} its, {1e3 * ms / max(1, st.iterations):7.1f} us/it, rel {st.final_relative_residual:.2e}")


if __name__ == "__main__":
    main()
