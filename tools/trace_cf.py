"""Kernel timeline of one batched CF split of every level (CUPTI via
torch.profiler): span, busy time and the gaps between consecutive kernels --
whether the split of the small levels is bound by the device chain or by
the host's launch rate. python tools/trace_cf.py [config]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

CFG = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = airg.Context(0)
p = problems.make(CFG)
prm = problems.setup_params(CFG)
h = airg.setup(airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx),
               ctx=ctx, **prm)
mats = [h.matrix_handle(l, 0) for l in range(h.n_levels)]
seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(h.n_levels)]
labs = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]
for _ in range(3):
    airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
    torch.cuda.synchronize()
path = "gpurun_out/trace_cf.json"
prof.export_chrome_trace(path)
evs = json.load(open(path))["traceEvents"]
ev = sorted([e for e in evs if e.get("cat") == "kernel"], key=lambda e: e["ts"])
rt = sorted([e for e in evs if e.get("cat") == "cuda_runtime" and "Launch" in e.get("name", "")],
            key=lambda e: e["ts"])
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
busy = sum(e["dur"] for e in ev)
gaps = [ev[i + 1]["ts"] - (ev[i]["ts"] + ev[i]["dur"]) for i in range(len(ev) - 1)]
print(f"C{CFG}: {len(ev)} kernels, GPU span {span:.1f} us, busy {busy:.1f} us, "
      f"gaps median {np.median(gaps):.2f} p90 {np.percentile(gaps, 90):.2f} us")
if rt:
    host = rt[-1]["ts"] + rt[-1]["dur"] - rt[0]["ts"]
    print(f"host launch calls {len(rt)}: first->last {host:.1f} us, mean call {np.mean([e['dur'] for e in rt]):.2f} us")
    # how far the device lags the host: kernel start - its launch call end
    lag = [ev[i]["ts"] - (rt[i]["ts"] + rt[i]["dur"]) for i in range(min(len(ev), len(rt)))]
    print(f"kernel start - launch return: median {np.median(lag):.1f} us, last {lag[-1]:.1f} us")
t0 = ev[-12]["ts"]
for e in ev[-12:]:
    nm = e["name"].replace("(anonymous namespace)::", "")[:60]
    print(f"  +{e['ts'] - t0:8.1f} us  dur {e['dur']:7.1f}  grid {e.get('args', {}).get('grid', '')}  {nm}")
