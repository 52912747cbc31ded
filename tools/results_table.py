"""BASELINE.md §4 results: every config C0-C4 at full size.

  python tools/results_table.py gpu  > gpurun_out/results_gpu.json   (GPU box)
  python tools/results_table.py cpu  > profiles/results_cpu.json      (reference build, CPU)

GPU: CF split ms (all levels back to back, fused split, one sync), setup ms
(the fast mode's fused operators included), solve DOF/s in fast mode (the
bench's) and exact mode (Richardson; C0 and C4 with the outer GMRES(30) --
see tests/test_gpu_parity.py), its, level-0 SpMV % of HBM. CPU: the reference's own serial build (oracle/_ref):
setup, CF split summed over its levels, one solve -- at full size where the
serial setup fits in minutes, else on the stated bounded sample.
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2408_08262_b200 import problems  # noqa: E402

OUTER = {0: 1, 4: 1}  # configs solved with the outer GMRES


def gpu():
    import torch
    from paper_2408_08262_b200 import airg
    ctx = airg.Context(0)
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6556.2
    out = {}
    for cfg in range(5):
        p = problems.make(cfg)
        prm = dict(problems.setup_params(cfg), fused_smooths=2)  # the fast mode's operators in the setup
        a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
        dA = airg.DeviceCSR.upload(a, ctx)
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        h = airg.setup(dA, ctx=ctx, **prm)
        del h
        e0, e1 = ev(), ev()
        e0.record(ctx.stream)
        h = airg.setup(dA, ctx=ctx, **prm)
        e1.record(ctx.stream)
        e1.synchronize()
        setup_ms = e0.elapsed_time(e1)
        # CF split of every level back to back, one synchronisation (the bench's cf_split_ms)
        mats = [h.matrix_handle(l, 0) for l in range(h.n_levels)]
        seeds = [int(problems.mix(np.uint64(0), np.uint64(l))) for l in range(h.n_levels)]
        labs = [ctx.empty(max(m.dims()[0], 1), torch.uint8) for m in mats]
        cfs = []
        for rep in range(4):
            s0, s1 = ev(), ev()
            s0.record(ctx.stream)
            airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm["max_loops"], labels=labs, ctx=ctx)
            s1.record(ctx.stream)
            s1.synchronize()
            cfs.append(s0.elapsed_time(s1))
        cf = float(np.median(cfs[1:]))
        tb = ctx.to_device(p.b)
        tx = ctx.empty(p.n, torch.float64)
        def solve_ms(fast):
            sk = dict(coarse_iterations=prm["coarse_iterations"], outer=OUTER.get(cfg, 0), gmres_restart=30,
                      max_iterations=1000, fast=fast)
            h.solve_device(tb, tx, **sk)
            ts = []
            for _ in range(3):
                s0, s1 = ev(), ev()
                s0.record(ctx.stream)
                st, _ = h.solve_device(tb, tx, **sk)
                s1.record(ctx.stream)
                s1.synchronize()
                ts.append(s0.elapsed_time(s1))
            return float(np.median(ts)), st
        ms_exact, st_exact = solve_ms(0)
        ms, st = solve_ms(1)
        A0 = h.matrix_handle(0, 0)
        n0, _, nnz0 = A0.dims()
        xv = torch.rand(n0, dtype=torch.float64, device=ctx.tdev)
        yv = torch.empty_like(xv)
        for _ in range(3):
            airg.spmv_device(A0, xv, yv, ctx=ctx)
        s0, s1 = ev(), ev()
        s0.record(ctx.stream)
        for _ in range(20):
            airg.spmv_device(A0, xv, yv, ctx=ctx)
        s1.record(ctx.stream)
        s1.synchronize()
        spmv_gbs = (12 * nnz0 + 4 * (n0 + 1) + 16 * n0) / (s0.elapsed_time(s1) / 20 / 1e3) / 1e9
        out[f"C{cfg}"] = dict(n=int(p.n), nnz=int(p.nnz), levels=int(h.n_levels), cf_split_ms=cf,
                              setup_ms=setup_ms, solve_ms=ms, dofs=p.n / (ms / 1e3),
                              iterations=int(st.iterations), converged=bool(st.converged),
                              exact_solve_ms=ms_exact, exact_dofs=p.n / (ms_exact / 1e3),
                              exact_iterations=int(st_exact.iterations),
                              outer="gmres(30)" if OUTER.get(cfg) else "richardson",
                              spmv_hbm_frac=spmv_gbs / peak)
        del h, dA
        torch.cuda.empty_cache()
    print(json.dumps(out))


# bounded CPU samples where the serial setup of the full system takes too long
CPU_SCALE = {0: 1.0, 1: 1.0, 2: 0.5, 3: 0.25, 4: 0.5}


def cpu():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import refpy
    lib = refpy.ref()
    out = {}
    for cfg in range(5):
        sc = CPU_SCALE[cfg]
        p = problems.make(cfg, sc)
        prm = problems.setup_params(cfg)
        A = lib.mat_from_problem(p)
        t0 = time.perf_counter()
        h = refpy.setup(lib, A, **prm)
        setup_ms = 1e3 * (time.perf_counter() - t0)
        cf = 0.0
        for l in range(h.info().n_levels):
            Al = h.matrix(l, 0)
            seed = int(problems.mix(np.uint64(0), np.uint64(l)))
            t0 = time.perf_counter()
            refpy.cf_split(lib, Al, prm, seed)
            cf += 1e3 * (time.perf_counter() - t0)
        scfg = refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"], outer=OUTER.get(cfg, 0),
                                      gmres_restart=30, max_iterations=1000)
        solver = h
        if OUTER.get(cfg):  # the reference has Richardson only: GMRES from the C restatement
            port = refpy.port()
            solver = refpy.setup(port, port.mat_from_problem(p), **prm)
        t0 = time.perf_counter()
        x, st, _ = solver.solve(p.b, scfg)
        its, conv = int(st.iterations), bool(st.converged)
        ms = 1e3 * (time.perf_counter() - t0)
        out[f"C{cfg}"] = dict(scale=sc, n=int(p.n), cf_split_ms=cf, setup_ms=setup_ms, solve_ms=ms,
                              dofs=p.n / (ms / 1e3), iterations=its, converged=conv,
                              solver="C restatement gmres(30)" if OUTER.get(cfg) else "reference richardson")
        print(json.dumps({f"C{cfg}": out[f"C{cfg}"]}), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    {"gpu": gpu, "cpu": cpu}[sys.argv[1]]()
