"""Kernel timeline of the CF split on every level of the C2 hierarchy
(torch.profiler / CUPTI): per-kernel totals and per-level GPU span vs the
event-timed wall of each airg_cf_split call.

  python tools/trace_cf.py [--out gpurun_out/trace_cf.txt]
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
    ap.add_argument("--out", default="gpurun_out/trace_cf.txt")
    args = ap.parse_args()
    ctx = airg.Context(0)
    p = problems.make(args.config)
    prm = problems.setup_params(args.config)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    h = airg.setup(dA, ctx=ctx, **prm)
    L = h.n_levels
    mats = [h.matrix_handle(l, 0) for l in range(L)]
    seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(L)]

    labs = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]

    def run():  # all levels back to back, one synchronisation (the bench's cf_split_ms)
        airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
    run()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                            torch.profiler.ProfilerActivity.CPU]) as prof:
        run()
        torch.cuda.synchronize()
    path = os.path.splitext(args.out)[0] + ".json"
    prof.export_chrome_trace(path)
    evs = json.load(open(path))["traceEvents"]
    ev = sorted([e for e in evs if e.get("cat") == "kernel"], key=lambda e: e["ts"])
    mem = sorted([e for e in evs if e.get("cat") in ("gpu_memset", "gpu_memcpy")], key=lambda e: e["ts"])
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    import re
    for e in ev:
        nm = e["name"].replace("(anonymous namespace)::", "")
        mt = re.search(r"(\w+)(<[^()]*>)?\(", nm)
        k = (mt.group(1) + (mt.group(2) or "")).replace("airg::", "")[:40] if mt else nm[:40]
        tot[k] += e["dur"]
        cnt[k] += 1
    span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
    lines = [f"CF split of all {L} levels: {len(ev)} kernels, {len(mem)} memset/memcpy, GPU span {span:.1f} us, "
             f"kernel busy {sum(tot.values()):.1f} us"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k:40s} {cnt[k]:5d} {v:9.1f} us  mean {v / cnt[k]:.2f}")
    # per level: first kernel start to last kernel end of each level's kernels
    per = len(ev) // L
    lines.append(f"per level ({per} kernels each): n, nnz, GPU span us, kernel busy us")
    for l in range(L):
        seg = ev[l * per:(l + 1) * per]
        d = mats[l].dims()
        lines.append(f"{l:3d} {d[0]:9d} {d[2]:10d} {seg[-1]['ts'] + seg[-1]['dur'] - seg[0]['ts']:9.1f} "
                     f"{sum(e['dur'] for e in seg):9.1f}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
