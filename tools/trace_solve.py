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

# CUPTI does not see the kernels of conditional graph bodies: host-driven loop
os.environ.setdefault("AIRG_DEVLOOP", "0")
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default="gpurun_out/trace_summary.txt")
    ap.add_argument("--what", default="solve", choices=["solve", "setup"])
    ap.add_argument("--outer", type=int, default=0, help="1 = outer GMRES(30)")
    ap.add_argument("--max-its", type=int, default=200)
    ap.add_argument("--fast", type=int, default=0, help="1 = fast arithmetic mode (lane groups, FMA)")
    args = ap.parse_args()
    ctx = airg.Context(0)
    p = problems.make(args.config, args.scale)
    prm = problems.setup_params(args.config)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    h = airg.setup(dA, ctx=ctx, **prm)
    tb = ctx.to_device(p.b)
    tx = ctx.empty(p.n, torch.float64)
    sk = dict(coarse_iterations=prm["coarse_iterations"], outer=args.outer, max_iterations=args.max_its, fast=args.fast)
    for _ in range(3):
        h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()

    class _St:
        iterations = 0
    st = _St()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        if args.what == "setup":
            h2 = airg.setup(dA, ctx=ctx, **prm)
        else:
            st, _ = h.solve_device(tb, tx, **sk)
        torch.cuda.synchronize()
    path = os.path.splitext(args.out)[0] + ".json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    # marginal cost of a kernel on the dependency chain: end(k) - end(k-1)
    # (with PDL a kernel starts before its predecessor ends, so 'dur' overlaps)
    for i, e in enumerate(ev):
        e["marg"] = e["dur"] if i == 0 else (e["ts"] + e["dur"]) - (ev[i - 1]["ts"] + ev[i - 1]["dur"])
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    import re
    for e in ev:
        nm = e["name"].replace("(anonymous namespace)::", "")
        mt = re.search(r"(\w+)(<[^()]*>)?\(", nm)
        name = (mt.group(1) + (mt.group(2) or "")).replace("airg::", "")[:48] if mt else nm[:48]
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
    if args.what == "solve" and st.iterations > 2 and not args.outer:
        # per-level breakdown of one middle iteration (kernel order of
        # enqueue_vcycle: R_0..R_{L-1}, coarse (2 ci - 1), then per level
        # L-1..0: prolong, fres1, fupd, fres2, fupd, ..., then axpy, resid, sum)
        L = h.n_levels
        plan = h.fused_plan() if args.fast else {"one_pass": [False] * L, "coarse_composed": False}
        nco = 1 if plan["coarse_composed"] else 2 * prm["coarse_iterations"] - 1
        per_lvl = 2 if args.fast else 1 + 2 * 2
        per_it = L + nco + (sum(1 if o else per_lvl for o in plan["one_pass"]) if args.fast else L * per_lvl) + 3
        if any("k_loop_check" in e["name"] for e in ev):
            per_it += 1  # device-side convergence test (AIRG_DEVLOOP)
        first = 2  # dot_partials, reduce_partials (bnorm)
        it = min(5, st.iterations - 1)
        seq = ev[first + it * per_it: first + (it + 1) * per_it]
        lines.append(f"-- iteration {it}: {len(seq)} kernels, span "
                     f"{seq[-1]['ts'] + seq[-1]['dur'] - seq[0]['ts']:.1f} us")
        lines.append(f"{'lvl':>3} {'n':>8} {'nnzR':>9} {'R us':>7} {'GB/s':>6} | {'nnzAF':>9} {'fres1':>7} {'GB/s':>6}"
                     f" | {'nnzFF':>8} {'fres2':>6} | {'nnzQ':>8} {'fupd':>6} {'GB/s':>6} | {'prol':>5}")
        asc = seq[L + nco:]
        if args.fast:
            lines[-1] = lines[-1] + "  (fast fused: per level R | A_F P residual | W x-update; 1p = one-pass K)"
            lines.append(f"coarse: {nco} kernels, " + " ".join(f"{e['marg']:.1f}" for e in seq[L:L + nco]) + " us")
            lines.append(f"{'lvl':>3} {'n':>8} {'nnzR':>9} {'R us':>7} | {'nnzAFP':>9} {'fres':>6} {'GB/s':>6} | {'nnzWX':>9} {'xw':>6} {'GB/s':>6}")
            pos = 0
            rows = []
            for l in range(L - 1, -1, -1):
                info = h.level(l)
                af, wx = h.fused_nnz(l)
                if plan["one_pass"][l]:
                    k = h.matrix_handle(l, 9).dims()[2]
                    e = asc[pos]
                    pos += 1
                    bk = 12 * k + 4 * info.n_f + 8 * info.n_c + 8 * info.n_f + 16 * info.n
                    rows.append(f"{l:3d} {info.n:8d} {info.nnz_r:9d} {seq[l]['marg']:7.1f} | 1p K {k:9d} {e['marg']:6.1f} "
                                f"{bk / e['marg'] / 1e3:6.0f}")
                    continue
                blk = asc[pos:pos + 2]
                pos += 2
                bf = 12 * af + 4 * info.n_f + 8 * info.n_c + 8 * info.n_f + 8 * info.n_f
                bw = 12 * wx + 4 * info.n_f + 8 * info.n_f + 24 * info.n
                rows.append(f"{l:3d} {info.n:8d} {info.nnz_r:9d} {seq[l]['marg']:7.1f} | {af:9d} {blk[0]['marg']:6.1f} "
                            f"{bf / blk[0]['marg'] / 1e3:6.0f} | {wx:9d} {blk[1]['marg']:6.1f} {bw / blk[1]['marg'] / 1e3:6.0f}")
            lines.extend(reversed(rows))
            L = 0
        for l in range(L):
            info = h.level(l)
            r_us = seq[l]["marg"]
            blk = asc[(L - 1 - l) * 5:(L - l) * 5]
            nnz_af = info.nnz_ff + info.nnz_fc
            br = 12 * info.nnz_r + 4 * info.n_c + 16 * info.n_c + 8 * info.n
            baf = 12 * nnz_af + 4 * info.n_f + 8 * info.n + 32 * info.n_f
            bq = 12 * info.nnz_ffinv + 4 * info.n_f + 24 * info.n_f
            lines.append(f"{l:3d} {info.n:8d} {info.nnz_r:9d} {r_us:7.1f} {br / r_us / 1e3:6.0f} | {nnz_af:9d} "
                         f"{blk[1]['marg']:7.1f} {baf / blk[1]['marg'] / 1e3:6.0f} | {info.nnz_ff:8d} "
                         f"{blk[3]['marg']:6.1f} | {info.nnz_ffinv:8d} {blk[2]['marg']:6.1f} "
                         f"{bq / blk[2]['marg'] / 1e3:6.0f} | {blk[0]['marg']:5.1f}")
        lines.append("(per-kernel columns are marginal times on the chain: end(k) - end(k-1))")
    if args.what == "setup":
        # one line per SpGEMM call: rows (grid of spgemm_bound x 256) and the
        # device time of each of its kernels, in call order
        calls = []
        for e in ev:
            nm = e["name"]
            if "spgemm_bound" in nm:
                calls.append({"rows~": e.get("args", {}).get("grid", [0])[0] * 256, "ts": e["ts"], "k": []})
            elif "spgemm" in nm and calls:
                mt = re.search(r"(spgemm_\w+)(<[^()]*>)?\(", nm.replace("(anonymous namespace)::", ""))
                calls[-1]["k"].append((mt.group(1) + (mt.group(2) or "") if mt else nm[:30], e["dur"]))
        lines.append("-- SpGEMM calls: rows~, total us, kernels")
        for i, c_ in enumerate(calls):
            tot_us = sum(d for _, d in c_["k"])
            lines.append(f"{i:3d} {c_['rows~']:9d} {tot_us:9.1f}  " + " ".join(f"{k}={d:.0f}" for k, d in c_["k"]))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
