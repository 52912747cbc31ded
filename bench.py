#!/usr/bin/env python
"""AIRG benchmark (driver contract: one JSON line from rank 0).

Workload (BASELINE.json configs[2], the largest structured single-GPU case):
3D 7-point upwind streaming operator, 128^3 cells = 2,097,152 unknowns,
fp64, alpha 0.5, DDC 0.1, poly order 4, truncation at 5,000 rows, coarse
poly order 8, Richardson to rtol 1e-10 from x = 0. Synthetic seeded input
(problems.py; no dataset exists for this operator).

One STEP = one complete AIRG solve (Richardson, V(0,2) cycles) of that
system with b already resident in HBM; value = unknowns solved per second
over all ranks. The hierarchy is built once before timing (setup time and
the CF-split time are reported alongside as setup_ms / cf_split_ms).
L2 is flushed (512 MiB write) before every timed step; the hierarchy
(~1.8 GB) is larger than L2 as well.

--impl reference times the reference's own serial CPU implementation
(oracle/_ref built from /root/reference, else the C restatement) on the
same configuration; each step is one full Richardson solve.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS_FILE = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def spmv_bytes(rows, cols, nnz):
    """int32 column + fp64 value per nonzero, int32 row
    pointer, x read once, y written once."""
    return 12 * nnz + 4 * (rows + 1) + 8 * cols + 8 * rows


def solve_alg_bytes(h, iterations, coarse_iterations, up_smooths=2):
    """Algorithmic HBM bytes of one solve: every operator the V-cycle applies
    is read once per application (12 B per nonzero + 4 B per row pointer) and
    every vector it needs is read or written once (8 B per entry, 4 B per
    index map entry). Per level (solve.cpp:93-146): R b; the first F-smooth's
    residual over A's F rows (A_ff and A_fc entries: nnz_ff + nnz_fc) with x,
    b_F, r_F and the kept A_fc x_C; Aff^-1 r_F with the x_F update (twice);
    the second residual over A_ff; the one-point prolongation. Per Richardson
    iteration the top residual r = b - A x with its norm and x += e; the
    coarse grid's polynomial iterations. The reference's unfused operator
    sequence (separate gathers, A_ff / A_fc SpMVs, vector temporaries) moves
    more; that count is reported separately (reference_op_bytes)."""
    info = h.info()
    per_cycle = 0
    for l in range(info.n_levels):
        lv = h.level(l)
        n, nf, nc = lv.n, lv.n_f, lv.n_c
        r = 12 * lv.nnz_r + 4 * (nc + 1) + 8 * n + 8 * nc
        fres1 = 12 * (lv.nnz_ff + lv.nnz_fc) + 4 * (nf + 1) + 8 * n + nf * (4 + 8 + 8 + 8)
        fupd = 12 * lv.nnz_ffinv + 4 * (nf + 1) + 8 * nf + nf * (4 + 16)
        fres2 = 12 * lv.nnz_ff + 4 * (nf + 1) + 8 * nf + nf * (4 + 8 + 8 + 8)
        prol = n * (4 + 8) + 8 * nc
        smooths = fres1 + fupd + (up_smooths - 1) * (fres2 + fupd)
        per_cycle += r + prol + smooths
    cn = info.coarse_n
    for it in range(coarse_iterations):
        per_cycle += 12 * info.coarse_inv_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
        if it:
            per_cycle += 12 * info.coarse_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
    top = h.level(0) if info.n_levels else None
    n0 = top.n if top else cn
    nnz0 = top.nnz if top else info.coarse_nnz
    resid = spmv_bytes(n0, n0, nnz0) + 8 * n0  # + b
    per_iter = per_cycle + resid + 24 * n0
    return iterations * per_iter + resid


def reference_op_bytes(h, iterations, coarse_iterations, up_smooths=2):
    """The same solve counted over the reference's unfused operations
    (every SpMV and vector op solve.cpp:34-259 issues,
    separately: x_F / x_C gathers, A_ff and A_fc SpMVs, b_F - . - ., scatter)."""
    info = h.info()
    per_cycle = 0
    for l in range(info.n_levels):
        lv = h.level(l)
        n, nf, nc = lv.n, lv.n_f, lv.n_c
        b = spmv_bytes(nc, n, lv.nnz_r) + spmv_bytes(n, nc, lv.nnz_p) + 24 * n
        smooth = (16 * nf + 16 * nc + spmv_bytes(nf, nf, lv.nnz_ff) + spmv_bytes(nf, nc, lv.nnz_fc)
                  + 16 * nf + 32 * nf + spmv_bytes(nf, nf, lv.nnz_ffinv) + 28 * nf)
        per_cycle += b + up_smooths * smooth
    cn = info.coarse_n
    for it in range(coarse_iterations):
        per_cycle += spmv_bytes(cn, cn, info.coarse_inv_nnz) + 24 * cn
        if it:
            per_cycle += spmv_bytes(cn, cn, info.coarse_nnz) + 24 * cn
    top = h.level(0) if info.n_levels else None
    n0 = top.n if top else cn
    nnz0 = top.nnz if top else info.coarse_nnz
    per_iter = per_cycle + spmv_bytes(n0, n0, nnz0) + 24 * n0 + 8 * n0 + 24 * n0
    return iterations * per_iter + spmv_bytes(n0, n0, nnz0) + 32 * n0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append(dict(sm=float(f[1]), smax=float(f[2]), hw=f[5], hwt=f[6], swt=f[7], pcap=f[8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = set()
        for r in rows:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                            ("swt", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in rows), "sm_max_mhz": max(r["smax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_lib():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import refpy  # cpu_baseline / reference arm only
    ref = None
    if os.path.exists(os.path.join(REPO, "oracle", "_ref", "libairgraph_ref.so")):
        ref = refpy.ref()
    return refpy, (ref if ref is not None else refpy.port()), ("reference" if ref is not None else "port")


def cpu_solve_sample(cfg_idx: int, nx: int):
    """Bounded CPU sample: the reference (or its restatement) on the same
    generator at nx^3, setup untimed, one Richardson solve timed."""
    from paper_2408_08262_b200 import problems
    refpy, lib, kind = oracle_lib()
    p = problems.c2_structured_3d(nx)
    prm = problems.setup_params(cfg_idx)
    A = lib.mat_from_problem(p)
    h = refpy.setup(lib, A, **prm)
    t0 = time.perf_counter()
    x, st, _ = h.solve(p.b, refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"]))
    t = time.perf_counter() - t0
    return {"value": p.n / t, "unit": "DOF/s", "cores": 1, "kind": kind,
            "sample": f"C2 generator at {nx}^3 ({p.n} unknowns): one serial Richardson solve "
                      f"({st.iterations} its, {t:.2f} s; setup untimed) on {cpu_model()}"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2408_08262_b200 import problems
    refpy, lib, kind = oracle_lib()
    # A bounded sample of the workload: the reference's serial setup of the
    # full 128^3 system alone takes ~150 s (one solve ~12 s, 0.18 M DOF/s,
    # measured in this container), so each step is one full Richardson solve
    # of the same C2 generator at --cpu-nx^3 (default 64^3: setup ~15 s once,
    # ~0.5 s per solve); DOF/s is size-normalised, and the smaller sample is
    # the reference's faster (cache-resident) case.
    full = problems.make(args.config, args.scale)
    if args.config == 2 and args.cpu_nx and args.cpu_nx < round(128 * args.scale):
        p = problems.c2_structured_3d(args.cpu_nx)
        sample = f"C2 generator at {args.cpu_nx}^3 ({p.n} unknowns) as a bounded sample of the {full.n}-unknown workload"
    else:
        p = full
        sample = "full workload"
    prm = problems.setup_params(args.config)
    A = lib.mat_from_problem(p)
    t0 = time.perf_counter()
    h = refpy.setup(lib, A, **prm)
    setup_s = time.perf_counter() - t0
    scfg = refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"])
    for _ in range(args.warmup):
        h.solve(p.b, scfg)
    times = []
    its = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        x, st, _ = h.solve(p.b, scfg)
        times.append(time.perf_counter() - t0)
        its = st.iterations
    tot = sum(times)
    value = p.n * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, full, "serial CPU"),
        "iterations": its, "final_relative_residual": st.final_relative_residual,
        "setup_ms": 1e3 * setup_s,
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": 1, "kind": kind,
                         "sample": f"{sample}, one Richardson solve per step on {cpu_model()} "
                                   f"(serial reference; {cpu_cores()} cores visible)"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "AIRG solve DOFs/s (Richardson to rtol 1e-10, V(0,2) cycles)"


def config_dict(args, p, par):
    names = {0: "C0 2D structured upwind 128^2", 1: "C1 2D unstructured upwind 512^2 quads",
             2: "C2 3D structured 7-point upwind 128^3", 3: "C3 2D S_n 256^2 x 64 angles",
             4: "C4 3D unstructured tets 2M/GPU"}
    return {"workload": names.get(args.config, str(args.config)) + (f" (scale {args.scale})" if args.scale != 1 else ""),
            "unknowns": int(p.n), "nnz": int(p.nnz), "alpha": 0.5, "ddc_fraction": 0.1, "poly_order": 4,
            "parallelism": par, "l2": "flushed (512 MiB write) before each timed step; hierarchy > L2"}


def run_gpu_dist(args):
    """N > 1 (torchrun, one process per GPU): weak scaling of the C2 family
    (128 x 128 x 128N cells, one 128^3 z-slab = 2,097,152 unknowns per GPU).
    The setup's row work is split over the ranks and all-gathered
    (airg_dist_setup: every rank holds the hierarchy), then every rank keeps
    its row slabs (z-slabs on level 0, the replay halving rule on coarser
    levels, the coarsest grid gathered on rank 0) and runs the distributed
    Richardson solve with NCCL halo exchanges and allreduced norms."""
    import torch
    import torch.distributed as dist
    from paper_2408_08262_b200 import airg, problems

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = airg.Context(local)
    stream = ctx.stream
    p = problems.c2_structured_3d(128, nz_slabs=ws)
    prm = problems.setup_params(2)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    uid = [airg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = airg.NcclComm(ws, rank, uid[0])
    # distributed setup: row work split over the ranks, slabs all-gathered
    # (airg_dist_setup); warmed once, then timed (max over ranks)
    del_h = airg.setup(dA, ctx=ctx, nranks=ws, rank=rank, comm=comm, **prm)
    del del_h
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h = airg.setup(dA, ctx=ctx, nranks=ws, rank=rank, comm=comm, **prm)
    e1.record(stream)
    e1.synchronize()
    setup_ms = e0.elapsed_time(e1)
    tsm = torch.tensor([setup_ms], device=ctx.tdev, dtype=torch.float64)
    dist.all_reduce(tsm, op=dist.ReduceOp.MAX)
    setup_ms = float(tsm[0])
    slab = p.n // ws
    starts = np.arange(ws + 1, dtype=np.int64) * slab
    d = airg.Dist(h, ws, rank=rank, comm=comm, threshold=2.0, starts=starts)
    lo, hi = starts[rank], starts[rank + 1]
    # CF split at N GPUs: the row-slab PMISR-DDC (airg_dist_cf_split) on
    # every level's operator with that level's slabs; max over ranks
    cf_ms = 0.0
    for l in range(h.n_levels):
        Al = h.matrix_handle(l, 0)
        sl = d.level_info(l)["starts"]
        seed = int(problems.mix(np.uint64(0), np.uint64(l)))
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        airg.dist_cf_split_device(Al, sl, rank=rank, comm=comm, alpha=prm["strength_alpha"],
                                  max_loops=prm["max_loops"], seed=seed, ctx=ctx)
        c1.record(stream)
        c1.synchronize()
        cf_ms += c0.elapsed_time(c1)
    tcf = torch.tensor([cf_ms], device=ctx.tdev, dtype=torch.float64)
    dist.all_reduce(tcf, op=dist.ReduceOp.MAX)
    cf_ms = float(tcf[0])
    with torch.cuda.stream(stream):
        tb = torch.from_numpy(p.b[lo:hi].copy()).to(ctx.tdev)
        tx = torch.empty(hi - lo, dtype=torch.float64, device=ctx.tdev)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=ctx.tdev)
    sk = dict(coarse_iterations=prm["coarse_iterations"])
    for _ in range(args.warmup):
        st, _ = d.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    l0 = ctx.launches()
    clk = ClockSampler(local).__enter__()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        torch.cuda.synchronize()
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        st, _ = d.solve_device(tb, tx, **sk)
        s1.record(stream)
        s1.synchronize()
        times.append(s0.elapsed_time(s1))
    launches = ctx.launches() - l0
    # e2e: host slab in, host slab out
    hb = torch.from_numpy(p.b[lo:hi].copy()).pin_memory()
    hx = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
    e2e = []
    for k in range(args.warmup + args.steps):
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        with torch.cuda.stream(stream):
            tb.copy_(hb, non_blocking=True)
        d.solve_device(tb, tx, **sk)
        with torch.cuda.stream(stream):
            hx.copy_(tx, non_blocking=True)
        s1.record(stream)
        s1.synchronize()
        if k >= args.warmup:
            e2e.append(s0.elapsed_time(s1))
    clk.__exit__(None, None, None)
    t = torch.tensor([sum(times), sum(e2e) / len(e2e)], device=ctx.tdev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, e2e_ms = float(t[0]), float(t[1])
    value = p.n * args.steps / (tot_ms / 1e3)
    levels = [d.level_info(l) for l in range(h.n_levels + 1)]
    # roofline of the whole distributed solve step against the N GPUs' HBM
    peak, peak_kind = hbm_peak()
    step_bytes = solve_alg_bytes(h, int(st.iterations), prm["coarse_iterations"])
    step_ach = step_bytes / (tot_ms / args.steps / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": step_ach, "peak": peak * ws, "unit": "GB/s",
            "frac": step_ach / (peak * ws), "traffic": None, "peak_kind": peak_kind,
            "kernel": f"one distributed AIRG solve step over {ws} GPUs (all row kernels + halo exchanges)",
            "alg_bytes_per_step": step_bytes, "avg_step_ms": tot_ms / args.steps}
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 family 128 x 128 x {128 * ws} (one 128^3 z-slab per GPU)",
                   "unknowns": int(p.n), "nnz": int(p.nnz), "alpha": 0.5, "ddc_fraction": 0.1,
                   "poly_order": 4, "parallelism": f"row slabs x{ws} (NCCL halos, replay halving, "
                   "gathered coarse grid; setup row work split over GPUs)",
                   "l2": "flushed (512 MiB write) before each timed step"},
        "iterations": int(st.iterations), "final_relative_residual": float(st.final_relative_residual),
        "levels": int(h.n_levels), "setup_ms": setup_ms,
        "active_ranks": [lv["active"] for lv in levels],
        "e2e": {"value": p.n / (e2e_ms / 1e3), "unit": "DOF/s", "h2d_bytes_per_step": 8 * int(hi - lo),
                "d2h_bytes_per_step": 8 * int(hi - lo), "ms_per_step": e2e_ms},
        "gpu_launches": int(launches), "cf_split_ms": cf_ms,
        "roofline": roof,
        "clocks": clk.summary(), "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    del d, comm
    dist.destroy_process_group()
    return 0


def run_gpu(args):
    import torch
    from paper_2408_08262_b200 import airg, problems

    ws, rank, local = dist_env()
    if ws > 1 or args.force_dist:
        return run_gpu_dist(args)
    dev = local
    ctx = airg.Context(dev)
    stream = ctx.stream
    p = problems.make(args.config, args.scale)
    prm = problems.setup_params(args.config)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        return e

    # ---- setup (warm once, then time)
    h = airg.setup(dA, ctx=ctx, **prm)
    del h
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(stream)
    h = airg.setup(dA, ctx=ctx, **prm)
    e1.record(stream)
    e1.synchronize()
    setup_ms = e0.elapsed_time(e1)
    info = h.info()

    # ---- CF split time: strength + PMISR + extract + DDC on every level's A.
    # cf_ms: all levels enqueued back to back (airg_cf_split_batch, one
    # synchronisation); cf_ms_each: one airg_cf_split call (and readback)
    # per level, summed.
    mats = [h.matrix_handle(l, 0) for l in range(info.n_levels)]
    seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(info.n_levels)]
    cf_lab = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]
    cf_ms = cf_ms_each = 0.0
    for rep in range(2):
        s0, s1 = ev(), ev()
        s0.record(stream)
        _, cf_reps = airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"],
                                                labels=cf_lab, ctx=ctx)
        s1.record(stream)
        s1.synchronize()
        cf_ms = s0.elapsed_time(s1)
        tot = 0.0
        for l, Al in enumerate(mats):
            s0, s1 = ev(), ev()
            s0.record(stream)
            airg.cf_split_device(Al, prm["strength_alpha"], prm["max_loops"], seeds[l], labels=cf_lab[l], ctx=ctx)
            s1.record(stream)
            s1.synchronize()
            tot += s0.elapsed_time(s1)
        cf_ms_each = tot
    # SURVEY 8(d) CF-split bytes per level: 2(12 nnz + 4n) + 16|S| + 26n
    cf_bytes = 0
    for Al, rp in zip(mats, cf_reps):
        n_l, _, z_l = Al.dims()
        cf_bytes += 2 * (12 * z_l + 4 * n_l) + 16 * int(rp.s_nnz) + 26 * n_l
    for l in range(info.n_levels):  # the split re-derives the setup's labels (untimed check)
        if not np.array_equal(cf_lab[l][: mats[l].dims()[0]].cpu().numpy(), h.labels(l)):
            raise RuntimeError(f"CF split of level {l} differs from the hierarchy's labels")

    # ---- device-resident solve steps
    with torch.cuda.stream(stream):
        tb = torch.from_numpy(p.b).to(ctx.tdev)
        tx = torch.empty(p.n, dtype=torch.float64, device=ctx.tdev)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=ctx.tdev)
    torch.cuda.synchronize()
    sk = dict(coarse_iterations=prm["coarse_iterations"])
    for _ in range(args.warmup):
        st, _ = h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    times = []
    l0 = ctx.launches()
    clk = ClockSampler(dev).__enter__()
    if True:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            s0, s1 = ev(), ev()
            s0.record(stream)
            st, _ = h.solve_device(tb, tx, **sk)
            s1.record(stream)
            s1.synchronize()
            times.append(s0.elapsed_time(s1))
    launches = ctx.launches() - l0
    torch.cuda.synchronize()
    local_ms = sum(times)
    tot_ms = local_ms
    if ws > 1:
        t = torch.tensor([local_ms], device=ctx.tdev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = p.n * ws * args.steps / (tot_ms / 1e3)
    x = ctx.to_host(tx)
    rel = np.linalg.norm(p.b - airg.spmv(dA, x, ctx=ctx)) / np.linalg.norm(p.b)

    # ---- the same system under the outer GMRES(30) the north star names
    # (device-resident b; reported beside the Richardson headline)
    gm = None
    try:
        gk = dict(sk, outer=1, gmres_restart=30)
        h.solve_device(tb, tx, **gk)
        gt = []
        for _ in range(3):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            g0, g1 = ev(), ev()
            g0.record(stream)
            gst, _ = h.solve_device(tb, tx, **gk)
            g1.record(stream)
            g1.synchronize()
            gt.append(g0.elapsed_time(g1))
        gms = statistics.median(gt)
        gm = {"value": p.n * ws / (gms / 1e3), "unit": "DOF/s", "ms_per_step": gms,
              "iterations": int(gst.iterations), "final_relative_residual": float(gst.final_relative_residual),
              "restart": 30}
    except Exception as exc:  # keep the headline line
        gm = {"error": str(exc)[:200]}

    # ---- end-to-end through the reference-facing call (host b -> host x)
    hb = torch.from_numpy(p.b.copy()).pin_memory()
    hx = torch.empty(p.n, dtype=torch.float64).pin_memory()
    e2e_times = []
    for k in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        s0, s1 = ev(), ev()
        s0.record(stream)
        res = h.solve_host_ptr(hb.data_ptr(), hx.data_ptr(), **sk)
        s1.record(stream)
        s1.synchronize()
        if k >= args.warmup:
            e2e_times.append(s0.elapsed_time(s1))
    clk.__exit__(None, None, None)  # clocks sampled across the device and e2e timed loops
    e2e_ms = sum(e2e_times) / len(e2e_times)
    e2e_value = p.n * ws / (e2e_ms / 1e3)

    # ---- roofline. The unit is the whole solve step ("per
    # V-cycle and per solve: sum over every SpMV and vector op"), whose
    # kernels replay as one captured graph per Richardson iteration; no single
    # kernel owns more than ~30% of it (profiles/r1_solve_launches.txt). The
    # level-0 SpMV (the reference's top hot spot, sparse.cpp:185-201) is
    # reported beside it, timed alone.
    step_bytes = solve_alg_bytes(h, int(st.iterations), prm["coarse_iterations"])
    peak, peak_kind = hbm_peak()
    step_achieved = step_bytes / (ms_per_step / 1e3) / 1e9
    A0 = h.matrix_handle(0, 0) if info.n_levels else dA
    n0, _, nnz0 = A0.dims()
    alg_bytes = spmv_bytes(n0, n0, nnz0)
    with torch.cuda.stream(stream):
        xv = torch.rand(n0, dtype=torch.float64, device=ctx.tdev)
        yv = torch.empty(n0, dtype=torch.float64, device=ctx.tdev)
    # (a) back to back: A + x + y = alg_bytes > the 126 MB L2, so the
    # operands stream from HBM; (b) one launch after an L2 flush (includes
    # the launch latency of a ~30 us kernel)
    for _ in range(3):
        airg.spmv_device(A0, xv, yv, ctx=ctx)
    k0, k1 = ev(), ev()
    reps = 50
    k0.record(stream)
    for _ in range(reps):
        airg.spmv_device(A0, xv, yv, ctx=ctx)
    k1.record(stream)
    k1.synchronize()
    kern_ms = k0.elapsed_time(k1) / reps
    kt = []
    for _ in range(10):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        f0, f1 = ev(), ev()
        f0.record(stream)
        airg.spmv_device(A0, xv, yv, ctx=ctx)
        f1.record(stream)
        f1.synchronize()
        kt.append(f0.elapsed_time(f1))
    flushed_ms = statistics.median(kt)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    prof = {}
    pf = os.path.join(REPO, "profiles", "dram_bytes.json")
    if os.path.exists(pf):
        try:
            prof = json.load(open(pf))
        except Exception:
            prof = {}
    step_traffic = prof.get("solve_dram_bytes_per_step")
    spmv_traffic = prof.get("spmv_dram_bytes_per_launch")

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_solve_sample(args.config, args.cpu_nx)
        except Exception as exc:  # keep the GPU line even if the checker fails
            cpu = {"value": None, "unit": "DOF/s", "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, p, "replicas (one independent system per GPU)" if ws > 1 else "single GPU"),
        "iterations": int(st.iterations), "final_relative_residual": float(rel),
        "levels": int(info.n_levels), "operator_complexity": info.operator_complexity,
        "setup_ms": setup_ms, "cf_split_ms": cf_ms, "cf_split_ms_sync_each_level": cf_ms_each,
        "cf_split_roofline": {"bound": "hbm", "achieved": cf_bytes / (cf_ms / 1e3) / 1e9, "peak": peak,
                              "unit": "GB/s", "frac": cf_bytes / (cf_ms / 1e3) / 1e9 / peak,
                              "alg_bytes_all_levels": cf_bytes,
                              "traffic": prof.get("cf_split_dram_bytes_all_levels"),
                              "bytes_rule": "sum over levels of 2(12 nnz + 4n) + 16|S| + 26n (SURVEY 8d)"},
        "roofline": {"bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s",
                     "frac": step_achieved / peak, "traffic": step_traffic,
                     "kernel": "one AIRG solve step: the captured V-cycle graph of all row kernels, "
                               "replayed once per Richardson iteration",
                     "alg_bytes_per_step": step_bytes, "avg_step_ms": ms_per_step, "peak_kind": peak_kind,
                     "reference_op_bytes_per_step": reference_op_bytes(h, int(st.iterations),
                                                                       prm["coarse_iterations"]),
                     "top_spmv": {"kernel": "rows_thread on level-0 A (exact CSR SpMV, y = A x)",
                                  "achieved": achieved, "frac": achieved / peak, "traffic": spmv_traffic,
                                  "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": kern_ms,
                                  "timing": "50 back-to-back launches; A + x + y exceed the 126 MB L2",
                                  "flushed_single_launch_ms": flushed_ms,
                                  "flushed_single_launch_frac": alg_bytes / (flushed_ms / 1e3) / 1e9 / peak}},
        "e2e": {"value": e2e_value, "unit": "DOF/s", "h2d_bytes_per_step": 8 * p.n,
                "d2h_bytes_per_step": 8 * p.n, "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "gmres": gm,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="airg", choices=["airg", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu-nx", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the distributed (NCCL row-slab) path even on one rank")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "airg":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
