"""Host-side CUDA runtime calls of one C2 setup (torch.profiler CUPTI
runtime records): total time per API, to find what the host spends the
setup's gaps on. python tools/trace_setup_api.py"""
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

ctx = airg.Context(0)
p = problems.make(2)
prm = problems.setup_params(2)
dA = airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx)
h = airg.setup(dA, ctx=ctx, **prm)
del h
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    h = airg.setup(dA, ctx=ctx, **prm)
    torch.cuda.synchronize()
path = "gpurun_out/trace_setup_api.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
evs = json.load(open(path))["traceEvents"]
api = [e for e in evs if e.get("cat") == "cuda_runtime" or e.get("cat") == "cuda_driver"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in api:
    tot[e["name"]] += e.get("dur", 0)
    cnt[e["name"]] += 1
top = [e for e in evs if e.get("ph") == "X" and e.get("cat") in ("cpu_op", "python_function", "user_annotation")]
span = max(e["ts"] + e.get("dur", 0) for e in api) - min(e["ts"] for e in api)
print(f"runtime calls {len(api)}, span {span:.0f} us, in calls {sum(tot.values()):.0f} us")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{k:40s} {cnt[k]:6d} {v:10.1f} us  mean {v / cnt[k]:.2f}")
