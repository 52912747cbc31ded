"""Warm, non-serialised kernel timeline of one C2 solve via torch.profiler
(CUPTI activity records; no cache flushing, unlike ncu). Writes a per-kernel
summary (device time, count, mean) plus the idle gaps between consecutive
kernels to gpurun_out/trace_summary.txt.

  python tools/trace_solve.py [--config 2] [--scale 1.0]
"""
import argparse
import collections
import json
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
    ap.add_argument("--out", default="gpurun_out/trace_summary.txt")
    args = ap.parse_args()
    ctx = airg.Context(0)
    p = problems.make(args.config, args.scale)
    prm = problems.setup_params(args.config)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
    tb = ctx.to_device(p.b)
    tx = ctx.empty(p.n, torch.float64)
    sk = dict(coarse_iterations=prm["coarse_iterations"])
    for _ in range(3):
        h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        st, _ = h.solve_device(tb, tx, **sk)
        torch.cuda.synchronize()
    path = "/tmp/trace_solve.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for e in ev:
        name = e["name"].split("(")[0].split("::")[-1][:48]
        tot[name] += e["dur"]
        cnt[name] += 1
    span = (ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]) if ev else 0.0
    busy = sum(e["dur"] for e in ev)
    gaps = [ev[i + 1]["ts"] - (ev[i]["ts"] + ev[i]["dur"]) for i in range(len(ev) - 1)]
    lines = [f"kernels {len(ev)}  span {span:.1f} us  busy {busy:.1f} us  iterations {st.iterations}",
             f"gap us: median {np.median(gaps):.2f} mean {np.mean(gaps):.2f} p90 {np.percentile(gaps, 90):.2f}"
             if gaps else "no gaps"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k:48s} {cnt[k]:6d} {v:10.1f} us {100 * v / max(busy, 1e-9):5.1f}%  mean {v / cnt[k]:.2f}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
