"""Host-side CUDA runtime calls and kernels of one setup (SETUP_CONFIG, default 2;
fast-mode fused operators included) -- C2 setup originally (torch.profiler CUPTI
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
CFG = int(os.environ.get("SETUP_CONFIG", "2"))
p = problems.make(CFG)
prm = dict(problems.setup_params(CFG), fused_smooths=2)
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

ker = [e for e in evs if e.get("cat") == "kernel"]
kt = collections.defaultdict(float)
kc = collections.Counter()
for e in ker:
    nm = e["name"].replace("(anonymous namespace)::", "").replace("airg::", "").split("(")[0][:62]
    kt[nm] += e.get("dur", 0)
    kc[nm] += 1
kspan = max(e["ts"] + e.get("dur", 0) for e in ker) - min(e["ts"] for e in ker)
# busy = union of kernel intervals
iv = sorted((e["ts"], e["ts"] + e.get("dur", 0)) for e in ker)
busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
for s0, e0 in iv[1:]:
    if s0 > cur_e:
        busy += cur_e - cur_s
        cur_s, cur_e = s0, e0
    else:
        cur_e = max(cur_e, e0)
busy += cur_e - cur_s
mc = [e for e in evs if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
print(f"C{CFG}: kernels {len(ker)}, memcpy/memset {len(mc)}, GPU span {kspan:.0f} us, busy (union) {busy:.0f} us, "
      f"sum of kernel durations {sum(kt.values()):.0f} us")
for k, v in sorted(kt.items(), key=lambda x: -x[1])[:30]:
    print(f"{k:62s} {kc[k]:6d} {v:10.1f} us  mean {v / kc[k]:.2f}")
