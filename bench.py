#!/usr/bin/env python
"""AIRG benchmark (driver contract: one JSON line from rank 0).

Workload (BASELINE.json configs[4], the configuration the metric's 1/2/4/8
GPU weak scaling is quoted on): the 3D unstructured P0 upwind streaming
operator on a jittered tet lattice, 70 x 70 x 68 cubes x 6 tets =
1,999,200 unknowns per GPU (z-slabs at N > 1), fp64, alpha 0.5, DDC 0.1,
poly order 4, truncation at 5,000 rows, coarse poly order 8; solved to
rtol 1e-10 from x = 0 by the outer right-preconditioned GMRES(30) with one
AIRG V(0,2) cycle per iteration. (The reference's own Richardson diverges on
this system -- level-0 smoother growth 2.33 on the best of its six fits --
so both arms run the same GMRES(30); tests/golden/full/c4.npz.)
Synthetic seeded input (problems.py; no dataset exists for this operator).

One STEP = one complete solve of that system with b already resident in HBM;
value = unknowns solved per second over all ranks. The hierarchy is built
once before timing (setup and CF-split times are reported alongside).
L2 is flushed (512 MiB write) before every timed step; the hierarchy
(~1 GB) and the Krylov basis (~1 GB) are larger than L2 as well.
`configs` adds C2 (128^3) and C3 (8.4 M unknowns) under Richardson, one GPU.

--impl reference times the reference's own CPU implementation (oracle/_ref
built from /root/reference; else the C restatement) on the SAME full-size
system with the same outer GMRES(30) around the reference's vcycle():
K full solves spread over all host cores (the reference is serial; its
solves of one hierarchy are reentrant, solve.hpp / SPEC.md:92).
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


def vcycle_alg_bytes(h, coarse_iterations, up_smooths=2, fast=False):
    """Algorithmic HBM bytes of one V-cycle (see solve_alg_bytes). fast: the
    fused ascent (fused.cu) -- per level R b, r1 = b_F - (A_F P) e_c and
    x = P e_c + W r1 (W rows on the F points, the C points prolongated)."""
    info = h.info()
    per_cycle = 0
    plan = h.fused_plan() if fast else None
    if fast:
        for l in range(info.n_levels):
            lv = h.level(l)
            n, nf, nc = lv.n, lv.n_f, lv.n_c
            afp, wx = h.fused_nnz(l)
            if plan["one_pass"][l]:
                # [b_{l+1}; y] = [R; W E_F^T] b_l, then x_F = y + K e_c (+ the C points)
                k = h.matrix_handle(l, 9).dims()[2]
                desc = 12 * (lv.nnz_r + wx) + 4 * (nc + nf + 1) + 8 * n + 8 * (nc + nf)
                asc = 12 * k + 4 * (nf + 1) + 8 * nc + nf * (4 + 8 + 8) + nc * (4 + 4 + 8)
                per_cycle += desc + asc
                continue
            r = 12 * lv.nnz_r + 4 * (nc + 1) + 8 * n + 8 * nc
            fres = 12 * afp + 4 * (nf + 1) + 8 * nc + nf * (4 + 8 + 8)
            xw = 12 * wx + 4 * (nf + 1) + 8 * nf + n * (4 + 4 + 8) + 8 * nc
            per_cycle += r + fres + xw
    # exact (reference-structured) V-cycle, per level (solve.cpp:93-146): R b;
    # the first F-smooth's residual over A's F rows (nnz_ff + nnz_fc) with x,
    # b_F, r_F and the kept A_fc x_C; Aff^-1 r_F with the x_F update (twice);
    # the second residual over A_ff; the one-point prolongation
    for l in range(0 if fast else info.n_levels):
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
    if fast and plan["coarse_composed"]:  # e = E_k b (fused.cu)
        return per_cycle + 12 * h.matrix_handle(info.n_levels, 9).dims()[2] + 4 * (cn + 1) + 16 * cn
    for it in range(coarse_iterations):
        per_cycle += 12 * info.coarse_inv_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
        if it:
            per_cycle += 12 * info.coarse_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
    return per_cycle


class OwnedView:
    """The hierarchy report of an owned distribution (airg_dist_report) in
    the shape vcycle_alg_bytes / gmres_alg_bytes read."""

    def __init__(self, d):
        self.d = d
        self.n_levels = d.n_levels

    def level(self, l):
        return self.d.report(l)

    def fused_nnz(self, l):
        return self.d.fused_nnz(l)

    def coarse_e_nnz(self):
        return self.d.coarse_e_nnz()

    def info(self):
        from types import SimpleNamespace
        c = self.d.report(self.d.n_levels)
        return SimpleNamespace(n_levels=self.d.n_levels, coarse_n=c.n, coarse_nnz=c.nnz, coarse_inv_nnz=c.nnz_ffinv,
                               coarse_effective_order=c.effective_order, coarse_attempts=max(1, c.poly_attempts))


def dist_vcycle_alg_bytes(v, coarse_iterations, up_smooths=2, fast=False):
    """Algorithmic bytes of one distributed V-cycle (dist.cu enqueue_vcycle,
    summed over the ranks): exact -- the exact V-cycle's; fast -- per level
    R b, r1 = b_F - (A_F P) e_c, x = P e_c + [W r1 on the F rows] (no
    one-pass level), the composed coarse solve when the distribution uses it."""
    if not fast:
        return vcycle_alg_bytes(v, coarse_iterations, up_smooths, False)
    info = v.info()
    per_cycle = 0
    for l in range(info.n_levels):
        lv = v.level(l)
        n, nf, nc = lv.n, lv.n_f, lv.n_c
        afp, wx = v.fused_nnz(l)
        per_cycle += 12 * lv.nnz_r + 4 * (nc + 1) + 8 * n + 8 * nc           # R b
        per_cycle += 12 * afp + 4 * (nf + 1) + 8 * nc + nf * (4 + 8 + 8)      # r1
        per_cycle += 12 * wx + 4 * (nf + 1) + 8 * nf + n * (4 + 4 + 8) + 8 * nc  # x
    cn = info.coarse_n
    ce = v.coarse_e_nnz() if hasattr(v, "coarse_e_nnz") else -1
    if ce >= 0:
        return per_cycle + 12 * ce + 4 * (cn + 1) + 16 * cn
    for it in range(coarse_iterations):
        per_cycle += 12 * info.coarse_inv_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
        if it:
            per_cycle += 12 * info.coarse_nnz + 4 * (cn + 1) + 8 * cn + 16 * cn
    return per_cycle


def dist_gmres_alg_bytes(v, iterations, coarse_iterations, restart=30, up_smooths=2, fast=False):
    """Algorithmic bytes of one distributed GMRES(m) solve (dist.cu
    dist_gmres, summed over the ranks). Per Arnoldi step: the V-cycle, Z_j =
    z (copy), w = A z, two CGS passes (dots: V_0..V_j and w read; update: V
    and w read, w written), |w|, v_{j+1} = w / |w| into V and the V-cycle
    input. Per restart: x += Z y, r = b - A x and its norm."""
    info = v.info()
    top = v.level(0) if info.n_levels else None
    n = top.n if top else info.coarse_n
    nnz = top.nnz if top else info.coarse_nnz
    cyc = dist_vcycle_alg_bytes(v, coarse_iterations, up_smooths, fast)
    spmv = spmv_bytes(n, n, nnz)
    tot = 8 * n
    left = iterations
    while left > 0:
        j_max = min(restart, left)
        for j in range(j_max):
            tot += cyc + 16 * n + spmv + 4 * (j + 1) * 8 * n + (2 + 4 + 1 + 3) * 8 * n
        tot += (j_max + 2) * 8 * n + spmv + 8 * n
        left -= j_max
    return tot


def gmres_alg_bytes(h, iterations, coarse_iterations, restart=30, up_smooths=2, fast=False):
    """Algorithmic HBM bytes of one GMRES(m) solve. Per Arnoldi step j (one
    outer iteration): the V-cycle (vcycle_alg_bytes), w = A z (SpMV + z
    written), classical Gram-Schmidt twice -- exact mode: three sweeps over
    V_0..V_j (dots; first update fused with the second dots; second update
    with the norm); fast mode: two (dots with w and v_j; the update with the
    Gram-corrected coefficients and the norm) -- plus w read / written per
    sweep, and v_{j+1} = w / |w| (exact); the fast mode's second sweep writes
    the unnormalised v_{j+1} and the V-cycle input instead (solve.cu
    GmPieces::step). Per restart: x += Z y (j + 2 vectors), r = b - A x and
    its norm."""
    info = h.info()
    top = h.level(0) if info.n_levels else None
    n = top.n if top else info.coarse_n
    nnz = top.nnz if top else info.coarse_nnz
    cyc = vcycle_alg_bytes(h, coarse_iterations, up_smooths, fast)
    spmv = spmv_bytes(n, n, nnz)
    tot = 8 * n  # ||b||
    left = iterations
    while left > 0:
        j_max = min(restart, left)
        for j in range(j_max):
            if fast:  # two sweeps: w read twice, v_{j+1} and the V-cycle input written
                tot += cyc + spmv + 8 * n + 2 * (j + 1) * 8 * n + 4 * 8 * n
            else:  # three sweeps, then v_{j+1} = w / |w| (w read, two vectors written)
                tot += cyc + spmv + 8 * n + 3 * (j + 1) * 8 * n + 5 * 8 * n + 24 * n
        tot += (j_max + 2) * 8 * n + spmv + 8 * n
        left -= j_max
    return tot


def solve_alg_bytes(h, iterations, coarse_iterations, up_smooths=2, fast=False):
    """Algorithmic HBM bytes of one Richardson solve: every operator the
    V-cycle applies is read once per application (12 B per nonzero + 4 B per
    row pointer) and every vector it needs is read or written once (8 B per
    entry, 4 B per index map entry) -- vcycle_alg_bytes; per iteration the top
    residual r = b - A x with its norm and x += e."""
    info = h.info()
    per_cycle = vcycle_alg_bytes(h, coarse_iterations, up_smooths, fast)
    top = h.level(0) if info.n_levels else None
    n0 = top.n if top else info.coarse_n
    nnz0 = top.nnz if top else info.coarse_nnz
    resid = spmv_bytes(n0, n0, nnz0) + 8 * n0  # + b
    per_iter = per_cycle + resid + 24 * n0
    return iterations * per_iter + resid


def csr_bytes(rows, nnz):
    """One CSR operand read or written once: int32 column + fp64 value per
    nonzero, int32 row pointer."""
    return 12 * nnz + 4 * (rows + 1)


def setup_alg_bytes(h, cf_bytes, poly_order, coarse_poly_order, fast):
    """Compulsory HBM bytes of one setup (air.cpp:285-410), the lower bound
    its time is quoted against: every operation reads each operand once and
    writes its result once (SpGEMMs and fixed-sparsity products: csr_bytes of
    the operands and of the result; SpMVs: spmv_bytes), intermediate products
    that never have to leave the chip (A P inside R (A P), W A_ff inside W_2)
    not counted. Per level: the CF split (SURVEY 8d rule, cf_bytes), the block
    extraction (A read, A_ff / A_fc / A_cf written), per fit attempt
    (poly_attempts) the power basis (poly_order SpMVs over A_ff, the Gram
    pass over its poly_order + 1 vectors), the fixed-sparsity assembly
    (effective_order - 1 products on A_ff's pattern: two reads and a write
    each, then the inverse written) and the growth guard (30 steps of
    u <- u - Q (A_ff u) with its norm, air.cpp:61-95); R = -A_cf Q + injection;
    the one-point P from A's rows; the Galerkin product R A P with the drop
    rule; fast mode: A_F P and W_2. Then the coarse fit."""
    info = h.info()
    total = cf_bytes
    for l in range(info.n_levels):
        L = h.level(l)
        nxt_n, nxt_nnz = ((h.level(l + 1).n, h.level(l + 1).nnz) if l + 1 < info.n_levels
                          else (info.coarse_n, info.coarse_nnz))
        aff = csr_bytes(L.n_f, L.nnz_ff)
        q = csr_bytes(L.n_f, L.nnz_ffinv)
        total += csr_bytes(L.n, L.nnz) + L.n + aff + csr_bytes(L.n_f, L.nnz_fc) + csr_bytes(L.n_c, L.nnz_cf)
        fit = poly_order * spmv_bytes(L.n_f, L.n_f, L.nnz_ff) + 8 * (poly_order + 1) * L.n_f
        fit += max(int(L.effective_order) - 1, 0) * 3 * aff + q
        fit += 30 * (spmv_bytes(L.n_f, L.n_f, L.nnz_ff) + spmv_bytes(L.n_f, L.n_f, L.nnz_ffinv) + 16 * L.n_f)
        total += int(L.poly_attempts) * fit
        total += csr_bytes(L.n_c, L.nnz_cf) + q + csr_bytes(L.n_c, L.nnz_r)             # R
        total += csr_bytes(L.n, L.nnz) + L.n + csr_bytes(L.n, L.nnz_p)                  # P
        total += (csr_bytes(L.n_c, L.nnz_r) + csr_bytes(L.n, L.nnz) + csr_bytes(L.n, L.nnz_p)
                  + csr_bytes(nxt_n, nxt_nnz))                                          # R A P
        if fast:
            afp, wx = h.fused_nnz(l)
            total += (csr_bytes(L.n_f, L.nnz_ff + L.nnz_fc) + csr_bytes(L.n, L.nnz_p) + csr_bytes(L.n_f, afp)
                      + 2 * q + aff + csr_bytes(L.n_f, wx))
    nc, zc, zq = info.coarse_n, info.coarse_nnz, info.coarse_inv_nnz
    cfit = coarse_poly_order * spmv_bytes(nc, nc, zc) + 8 * (coarse_poly_order + 1) * nc
    cfit += max(int(info.coarse_effective_order) - 1, 0) * 3 * csr_bytes(nc, zc) + csr_bytes(nc, zq)
    cfit += 30 * (spmv_bytes(nc, nc, zc) + spmv_bytes(nc, nc, zq) + 16 * nc)
    total += int(info.coarse_attempts) * cfit
    return int(total)


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


def solver_kw(cfg_idx: int) -> dict:
    """Outer solver per config: GMRES(30) for C0 (its config names it) and
    C4 (the reference's Richardson diverges there), Richardson otherwise."""
    return dict(outer=1, gmres_restart=30) if cfg_idx in (0, 4) else dict(outer=0)


def solver_name(cfg_idx: int) -> str:
    return "outer GMRES(30) + AIRG V(0,2)" if cfg_idx in (0, 4) else "Richardson + AIRG V(0,2)"


def cpu_solve_sample(cfg_idx: int):
    """Bounded CPU sample for `cpu_baseline`: the reference (or its
    restatement) on the same generator at half the linear size (1/8 of the
    unknowns; ~10 s of serial work), setup untimed, one solve timed with the
    same outer solver."""
    from paper_2408_08262_b200 import problems
    refpy, lib, kind = oracle_lib()
    p = problems.make(cfg_idx, 0.5)
    prm = problems.setup_params(cfg_idx)
    A = lib.mat_from_problem(p)
    h = refpy.setup(lib, A, **prm)
    t0 = time.perf_counter()
    x, st, _ = h.solve(p.b, refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"],
                                                   max_iterations=400, **solver_kw(cfg_idx)))
    t = time.perf_counter() - t0
    return {"value": p.n / t, "unit": "DOF/s", "cores": 1, "kind": kind,
            "sample": f"C{cfg_idx} generator at half linear size ({p.n} unknowns): one serial "
                      f"{solver_name(cfg_idx)} solve ({st.iterations} its, {t:.2f} s; setup untimed) "
                      f"on {cpu_model()}"}


def run_reference(args):
    """The reference's own serial CPU path on the SAME full-size system and
    outer solver as the GPU arm, with all host cores. The serial setup (~55 s
    for C4) runs once, untimed. One complete solve is then timed alone (its
    iteration count I and time are reported). For GMRES(m) each of the K
    steps is a bounded sample: one full restart cycle (m iterations from
    x = 0 -- the same work as every complete cycle of the solve), the K
    samples running concurrently on min(K, cores) threads (the reference's
    solves of one hierarchy are reentrant; ctypes releases the
    GIL); value = K * m / I solves' worth of unknowns over the pool's wall
    time. For Richardson each step is one complete solve."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from concurrent.futures import ThreadPoolExecutor
    from paper_2408_08262_b200 import problems
    refpy, lib, kind = oracle_lib()
    p = problems.make(args.config, args.scale)
    prm = problems.setup_params(args.config)
    A = lib.mat_from_problem(p)
    t0 = time.perf_counter()
    h = refpy.setup(lib, A, **prm)
    setup_s = time.perf_counter() - t0
    skw = solver_kw(args.config)
    full_cfg = refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"], max_iterations=400, **skw)
    t0 = time.perf_counter()
    _, fst, _ = h.solve(p.b, full_cfg)
    full_s = time.perf_counter() - t0
    its = int(fst.iterations)
    gm = skw["outer"] == 1
    m = skw.get("gmres_restart", 30)
    step_cfg = (refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"], max_iterations=min(m, its), **skw)
                if gm else full_cfg)
    frac = min(m, its) / its if gm else 1.0  # one step = this fraction of a complete solve
    threads = max(1, min(args.steps, cpu_cores()))

    def one(_):
        t = time.perf_counter()
        h.solve(p.b, step_cfg)
        return time.perf_counter() - t

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        res = list(pool.map(one, range(args.steps)))
    wall = time.perf_counter() - t0
    solves = args.steps * frac
    value = p.n * solves / wall
    sample = (f"full workload ({p.n} unknowns): one complete {solver_name(args.config)} solve timed alone "
              f"({its} its, {full_s:.1f} s), then {args.steps} samples of one full GMRES({m}) restart cycle "
              f"({min(m, its)} iterations from x = 0 = {frac:.3f} of a solve) on {threads} concurrent threads"
              if gm else f"full workload ({p.n} unknowns): {args.steps} complete {solver_name(args.config)} "
                         f"solves on {threads} concurrent threads")
    sample += f" of {cpu_model()} ({cpu_cores()} cores visible); setup once, untimed"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, p, f"serial reference x {threads} concurrent solves"),
        "iterations": its, "final_relative_residual": float(fst.final_relative_residual),
        "converged": bool(fst.converged), "setup_ms": 1e3 * setup_s,
        "single_solve_ms": 1e3 * full_s, "single_solve_dof_s": p.n / full_s,
        "step_ms_mean": 1e3 * sum(res) / len(res),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "AIRG solve DOFs/s"


CONFIG_NAMES = {0: "C0 2D structured upwind 128^2", 1: "C1 2D unstructured upwind 512^2 quads",
                2: "C2 3D structured 7-point upwind 128^3", 3: "C3 2D S_n 256^2 x 64 angles",
                4: "C4 3D unstructured tets, 70x70x68 cubes x 6 = 1,999,200 tets per GPU"}


def config_dict(args, p, par, cfg_idx=None):
    c = args.config if cfg_idx is None else cfg_idx
    return {"workload": CONFIG_NAMES.get(c, str(c)) + (f" (scale {args.scale})" if args.scale != 1 else ""),
            "unknowns": int(p.n), "nnz": int(p.nnz), "alpha": 0.5, "ddc_fraction": 0.1, "poly_order": 4,
            "solver": solver_name(c) + " to rtol 1e-10 from x = 0",
            "parallelism": par, "l2": "flushed (512 MiB write) before each timed step; hierarchy > L2"}


def run_gpu_dist(args):
    """N > 1 (torchrun, one process per GPU): weak scaling of the metric's
    config C4 -- a 70 x 70 x 68N cube lattice split into z-slabs of 68 cube
    layers (1,999,200 tets) per GPU, as BASELINE configs[4] states. Each rank
    generates its own slab (global column indices) and the owned-row
    distributed setup (airg_dist_setup_owned) builds every level with each
    rank holding only its rows (CF split on the slabs, halo rows of A_ff,
    Aff^-1 and A P fetched over NCCL, the replay halving rule on coarser
    levels, the coarsest grid gathered on rank 0). Then the distributed outer
    GMRES(30) around the row-slab V-cycle runs with NCCL halo exchanges and
    allreduced inner products."""
    import torch
    import torch.distributed as dist
    from paper_2408_08262_b200 import airg, problems

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = airg.Context(local)
    stream = ctx.stream
    dev = torch.device("cuda", local)
    nzl = round(68 * args.scale) if args.scale != 1 else 68
    nxy = round(70 * args.scale) if args.scale != 1 else 70
    ps = problems.c4_tets_3d(nxy, nxy, nzl, z0=nzl * rank, nz_total=nzl * ws)
    slab = ps.n
    N = slab * ws
    a_loc = airg.SparseMatrix.from_arrays(slab, N, ps.row_offsets, ps.cols, ps.vals)
    dA = airg.DeviceCSR.upload(a_loc, ctx)
    fast = args.mode == "fast"
    # fast mode: the fused level operators (A_F P, W_2) built on the slabs inside the timed setup
    prm = dict(problems.setup_params(4), fused_smooths=2 if fast else -1)
    uid = [airg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = airg.NcclComm(ws, rank, uid[0])
    starts = np.arange(ws + 1, dtype=np.int64) * slab
    lo, hi = starts[rank], starts[rank + 1]
    # owned setup, warmed once, then timed (max over ranks)
    warm = airg.Dist.setup_owned(dA, ws, rank=rank, comm=comm, threshold=2.0, starts=starts, ctx=ctx, **prm)
    del warm
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    d = airg.Dist.setup_owned(dA, ws, rank=rank, comm=comm, threshold=2.0, starts=starts, ctx=ctx, **prm)
    e1.record(stream)
    e1.synchronize()
    setup_ms = e0.elapsed_time(e1)
    cf_ms = d.setup_times()[1]  # device time of the setup's CF splits, all levels
    tsm = torch.tensor([setup_ms, cf_ms, float(d.rank_bytes())], device=ctx.tdev, dtype=torch.float64)
    dist.all_reduce(tsm, op=dist.ReduceOp.MAX)
    setup_ms, cf_ms, max_rank_bytes = float(tsm[0]), float(tsm[1]), float(tsm[2])
    with torch.cuda.stream(stream):
        tb = torch.from_numpy(ps.b.copy()).to(ctx.tdev)
        tx = torch.empty(hi - lo, dtype=torch.float64, device=ctx.tdev)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=ctx.tdev)
    sk = dict(coarse_iterations=prm["coarse_iterations"], max_iterations=400, fast=int(fast), **solver_kw(4))
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
    hb = torch.from_numpy(ps.b.copy()).pin_memory()
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
    value = N * args.steps / (tot_ms / 1e3)
    hv_ = OwnedView(d)
    levels = [d.level_info(l) for l in range(d.n_levels + 1)]
    # roofline of the whole distributed solve step against the N GPUs' HBM
    peak, peak_kind = hbm_peak()
    step_bytes = dist_gmres_alg_bytes(hv_, int(st.iterations), prm["coarse_iterations"], fast=fast)
    step_ach = step_bytes / (tot_ms / args.steps / 1e3) / 1e9
    # NVLink: halo bytes every process receives (exact, from the halo plans)
    # per V-cycle / level-0 SpMV, plus the allreduce payloads of the GMRES
    # inner products (2 (j + 1) + 1 doubles per step), summed over ranks
    hv, hs = d.halo_bytes(**sk)
    its_n = int(st.iterations)
    m = sk.get("gmres_restart", 30)
    ar = sum(8 * (2 * (k % m + 1) + 1) for k in range(its_n)) * (ws - 1) / max(1, ws) * 2
    mine = its_n * (hv + hs) + ((its_n + m - 1) // m + 1) * hs + ar
    tnv = torch.tensor([float(mine)], device=ctx.tdev, dtype=torch.float64)
    dist.all_reduce(tnv, op=dist.ReduceOp.SUM)
    nv_bytes = float(tnv[0])
    nv_ach = nv_bytes / ws / (tot_ms / args.steps / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": step_ach, "peak": peak * ws, "unit": "GB/s",
            "frac": step_ach / (peak * ws), "traffic": None, "peak_kind": peak_kind,
            "nvlink": {"bytes_per_step_all_ranks": nv_bytes, "achieved_per_gpu": nv_ach, "peak_per_gpu": 900.0,
                       "unit": "GB/s", "frac": nv_ach / 900.0,
                       "rule": "halo entries received per exchange x 8 B (dist.cu dist_halo_bytes) + ring "
                               "allreduce payloads of the GMRES inner products"},
            "kernel": f"one distributed AIRG solve step over {ws} GPUs (all row kernels + halo exchanges)",
            "alg_bytes_per_step": step_bytes, "avg_step_ms": tot_ms / args.steps}
    # setup against the N GPUs' HBM (the CF-split term without |S|: the owned
    # report does not carry the strength counts)
    cf_b = sum(2 * (12 * hv_.level(l).nnz + 4 * hv_.level(l).n) + 26 * hv_.level(l).n for l in range(d.n_levels))
    sb = setup_alg_bytes(hv_, cf_b, prm["poly_order"], prm["coarse_poly_order"], fast)
    setup_roof = {"bound": "hbm", "achieved": sb / (setup_ms / 1e3) / 1e9, "peak": peak * ws, "unit": "GB/s",
                  "frac": sb / (setup_ms / 1e3) / 1e9 / (peak * ws), "alg_bytes": sb,
                  "bytes_rule": "compulsory bytes of every setup operation, each operand read once and each "
                                "result written once (bench.py setup_alg_bytes)"}
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C4 3D unstructured tets, {nxy} x {nxy} x {nzl * ws} cubes x 6 "
                               f"(one {nzl}-layer z-slab = {ps.n} tets per GPU)",
                   "unknowns": int(N), "nnz": int(d.report(0).nnz), "alpha": 0.5, "ddc_fraction": 0.1,
                   "poly_order": 4, "solver": solver_name(4) + " to rtol 1e-10 from x = 0", "mode": args.mode,
                   "parallelism": f"row slabs x{ws} (NCCL halos and allreduces, replay halving, "
                   "gathered coarse grid; owned-row setup: every rank builds only its rows)",
                   "l2": "flushed (512 MiB write) before each timed step"},
        "iterations": int(st.iterations), "final_relative_residual": float(st.final_relative_residual),
        "levels": int(d.n_levels), "setup_ms": setup_ms,
        "active_ranks": [lv["active"] for lv in levels],
        "max_rank_solve_bytes": max_rank_bytes,
        "e2e": {"value": N / (e2e_ms / 1e3), "unit": "DOF/s", "h2d_bytes_per_step": 8 * int(hi - lo),
                "d2h_bytes_per_step": 8 * int(hi - lo), "ms_per_step": e2e_ms},
        "gpu_launches": int(launches), "cf_split_ms": cf_ms,
        "setup_roofline": setup_roof,
        "roofline": roof,
        "clocks": clk.summary(), "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    del d, comm
    dist.destroy_process_group()
    return 0


def _ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def time_solves(h, ctx, tb, tx, flush, steps, sk):
    """Device-resident solves, L2 flushed before each; per-step event times."""
    import torch
    stream = ctx.stream
    out = []
    st = None
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        s0, s1 = _ev(), _ev()
        s0.record(stream)
        st, _ = h.solve_device(tb, tx, **sk)
        s1.record(stream)
        s1.synchronize()
        out.append(s0.elapsed_time(s1))
    return out, st


def extra_config(ctx, cfg_idx, flush, fast, steps=5, warmup=3):
    """A secondary single-GPU line (C2 / C3): setup + device-resident solves."""
    import torch
    from paper_2408_08262_b200 import airg, problems
    p = problems.make(cfg_idx)
    prm = dict(problems.setup_params(cfg_idx), fused_smooths=2 if fast else -1)
    dA = airg.DeviceCSR.upload(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), ctx)
    h = airg.setup(dA, ctx=ctx, **prm)
    del h
    torch.cuda.synchronize()
    e0, e1 = _ev(), _ev()
    e0.record(ctx.stream)
    h = airg.setup(dA, ctx=ctx, **prm)
    e1.record(ctx.stream)
    e1.synchronize()
    setup_ms = e0.elapsed_time(e1)
    with torch.cuda.stream(ctx.stream):
        tb = torch.from_numpy(p.b).to(ctx.tdev)
        tx = torch.empty(p.n, dtype=torch.float64, device=ctx.tdev)
    sk = dict(coarse_iterations=prm["coarse_iterations"], max_iterations=400, fast=int(fast), **solver_kw(cfg_idx))
    for _ in range(warmup):
        h.solve_device(tb, tx, **sk)
    times, st = time_solves(h, ctx, tb, tx, flush, steps, sk)
    ms = sum(times) / len(times)
    its = int(st.iterations)
    byts = (gmres_alg_bytes(h, its, prm["coarse_iterations"], fast=fast) if sk["outer"]
            else solve_alg_bytes(h, its, prm["coarse_iterations"], fast=fast))
    peak, _ = hbm_peak()
    out = {"workload": CONFIG_NAMES[cfg_idx], "unknowns": int(p.n), "solver": solver_name(cfg_idx),
           "mode": "fast" if fast else "exact",
           "value": p.n / (ms / 1e3), "unit": "DOF/s", "ms_per_step": ms, "steps": steps,
           "iterations": its, "final_relative_residual": float(st.final_relative_residual),
           "levels": int(h.n_levels), "setup_ms": setup_ms,
           "roofline_frac": byts / (ms / 1e3) / 1e9 / peak}
    del h, dA
    return out


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
    fast = args.mode == "fast"
    # fast mode: the fused level operators are built inside the timed setup
    prm = dict(problems.setup_params(args.config), fused_smooths=2 if fast else -1)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    ev = _ev

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
    setup_bytes = setup_alg_bytes(h, cf_bytes, prm["poly_order"], prm["coarse_poly_order"], fast)
    for l in range(info.n_levels):  # the split re-derives the setup's labels (untimed check)
        if not np.array_equal(cf_lab[l][: mats[l].dims()[0]].cpu().numpy(), h.labels(l)):
            raise RuntimeError(f"CF split of level {l} differs from the hierarchy's labels")

    # ---- device-resident solve steps
    with torch.cuda.stream(stream):
        tb = torch.from_numpy(p.b).to(ctx.tdev)
        tx = torch.empty(p.n, dtype=torch.float64, device=ctx.tdev)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=ctx.tdev)
    torch.cuda.synchronize()
    sk = dict(coarse_iterations=prm["coarse_iterations"], max_iterations=400, fast=int(fast),
              **solver_kw(args.config))
    for _ in range(args.warmup):
        st, _ = h.solve_device(tb, tx, **sk)
    torch.cuda.synchronize()
    l0 = ctx.launches()
    clk = ClockSampler(dev).__enter__()
    times, st = time_solves(h, ctx, tb, tx, flush, args.steps, sk)
    launches = ctx.launches() - l0
    torch.cuda.synchronize()
    tot_ms = sum(times)
    ms_per_step = tot_ms / args.steps
    value = p.n * args.steps / (tot_ms / 1e3)
    x = ctx.to_host(tx)
    rel = np.linalg.norm(p.b - airg.spmv(dA, x, ctx=ctx)) / np.linalg.norm(p.b)

    # ---- end-to-end through the reference-facing call (host b -> host x)
    hb = torch.from_numpy(p.b.copy()).pin_memory()
    hx = torch.empty(p.n, dtype=torch.float64).pin_memory()
    e2e_times = []
    for k in range(args.warmup + args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        s0, s1 = ev(), ev()
        s0.record(stream)
        h.solve_host_ptr(hb.data_ptr(), hx.data_ptr(), **sk)
        s1.record(stream)
        s1.synchronize()
        if k >= args.warmup:
            e2e_times.append(s0.elapsed_time(s1))
    clk.__exit__(None, None, None)  # clocks sampled across the device and e2e timed loops
    e2e_ms = sum(e2e_times) / len(e2e_times)
    e2e_value = p.n / (e2e_ms / 1e3)
    # the other arithmetic mode on the same hierarchy (exact = the reference's bits)
    other = {}
    try:
        ok = dict(sk, fast=0 if fast else 1)
        for _ in range(2):
            h.solve_device(tb, tx, **ok)
        ot, ost = time_solves(h, ctx, tb, tx, flush, 3, ok)
        oms = sum(ot) / len(ot)
        other = {"mode": "exact" if fast else "fast", "value": p.n / (oms / 1e3), "unit": "DOF/s",
                 "ms_per_step": oms, "iterations": int(ost.iterations),
                 "final_relative_residual": float(ost.final_relative_residual)}
    except Exception as exc:
        other = {"error": str(exc)[:200]}

    # ---- roofline. The unit is the whole solve step ("per
    # V-cycle and per solve: sum over every SpMV and vector op"): no single
    # kernel owns more than ~15% of it (profiles/). The level-0 SpMV (the
    # reference's top hot spot, sparse.cpp:185-201) is reported beside it.
    its = int(st.iterations)
    step_bytes = (gmres_alg_bytes(h, its, prm["coarse_iterations"], fast=fast) if sk["outer"]
                  else solve_alg_bytes(h, its, prm["coarse_iterations"], fast=fast))
    peak, peak_kind = hbm_peak()
    step_achieved = step_bytes / (ms_per_step / 1e3) / 1e9
    A0 = h.matrix_handle(0, 0) if info.n_levels else dA
    n0, _, nnz0 = A0.dims()
    alg_bytes = spmv_bytes(n0, n0, nnz0)
    with torch.cuda.stream(stream):
        xv = torch.rand(n0, dtype=torch.float64, device=ctx.tdev)
        yv = torch.empty(n0, dtype=torch.float64, device=ctx.tdev)
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
    # time per V-cycle: the captured V-cycle graph through the
    # C-ABI (b copied in, x copied out: two n-vector device copies included)
    vk = dict(coarse_iterations=prm["coarse_iterations"], fast=int(fast))
    for _ in range(3):
        h.vcycle_device(xv, yv, **vk)
    k0.record(stream)
    for _ in range(20):
        h.vcycle_device(xv, yv, **vk)
    k1.record(stream)
    k1.synchronize()
    vcycle_ms = k0.elapsed_time(k1) / 20
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
    # the same after a clean flush: the 512 MiB write, then a 256 MiB read of
    # another buffer, so L2 holds clean lines and the flush's dirty lines are
    # not written back while the timed kernel runs
    with torch.cuda.stream(stream):
        rflush = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=ctx.tdev)
    kc = []
    for _ in range(10):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
            rsum = rflush.sum()
        f0, f1 = ev(), ev()
        f0.record(stream)
        airg.spmv_device(A0, xv, yv, ctx=ctx)
        f1.record(stream)
        f1.synchronize()
        kc.append(f0.elapsed_time(f1))
    del rsum, rflush
    clean_ms = statistics.median(kc)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    prof = {}
    pf = os.path.join(REPO, "profiles", "dram_bytes.json")
    if os.path.exists(pf):
        try:
            prof = json.load(open(pf)).get(f"C{args.config}", {})
        except Exception:
            prof = {}

    extras = {}
    if not args.no_extras and args.scale == 1:
        del h
        for c in (2, 3):
            if c == args.config:
                continue
            try:
                extras[f"C{c}"] = extra_config(ctx, c, flush, fast)
            except Exception as exc:  # keep the headline line
                extras[f"C{c}"] = {"error": str(exc)[:200]}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_solve_sample(args.config)
        except Exception as exc:  # keep the GPU line even if the checker fails
            cpu = {"value": None, "unit": "DOF/s", "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_dict(args, p, "single GPU"), mode=args.mode),
        "iterations": its, "final_relative_residual": float(rel),
        "other_mode": other,
        "levels": int(info.n_levels), "operator_complexity": info.operator_complexity,
        "vcycle_ms": vcycle_ms,
        "setup_ms": setup_ms, "cf_split_ms": cf_ms, "cf_split_ms_sync_each_level": cf_ms_each,
        "cf_split_roofline": {"bound": "hbm", "achieved": cf_bytes / (cf_ms / 1e3) / 1e9, "peak": peak,
                              "unit": "GB/s", "frac": cf_bytes / (cf_ms / 1e3) / 1e9 / peak,
                              "alg_bytes_all_levels": cf_bytes,
                              "traffic": prof.get("cf_split_dram_bytes_all_levels"),
                              "bytes_rule": "sum over levels of 2(12 nnz + 4n) + 16|S| + 26n (SURVEY 8d)"},
        "setup_roofline": {"bound": "hbm", "achieved": setup_bytes / (setup_ms / 1e3) / 1e9, "peak": peak,
                           "unit": "GB/s", "frac": setup_bytes / (setup_ms / 1e3) / 1e9 / peak,
                           "alg_bytes": setup_bytes,
                           "bytes_rule": "compulsory bytes of every setup operation, each operand read once and "
                                         "each result written once (bench.py setup_alg_bytes)"},
        "roofline": {"bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s",
                     "frac": step_achieved / peak, "traffic": prof.get("solve_dram_bytes_per_step"),
                     "kernel": "one AIRG solve step: every kernel of the solve (V-cycle graphs, "
                               "Krylov orthogonalisation, residuals)",
                     "alg_bytes_per_step": step_bytes, "avg_step_ms": ms_per_step, "peak_kind": peak_kind,
                     "top_spmv": {"kernel": "level-0 CSR SpMV y = A x",
                                  "achieved": achieved, "frac": achieved / peak,
                                  "traffic": prof.get("spmv_dram_bytes_per_launch"),
                                  "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": kern_ms,
                                  "timing": "50 back-to-back launches",
                                  "flushed_single_launch_ms": flushed_ms,
                                  "flushed_single_launch_frac": alg_bytes / (flushed_ms / 1e3) / 1e9 / peak,
                                  "clean_flushed_single_launch_ms": clean_ms,
                                  "clean_flushed_single_launch_frac": alg_bytes / (clean_ms / 1e3) / 1e9 / peak,
                                  "flush": "512 MiB write before each launch (dirty L2: its write-back overlaps "
                                           "the launch); clean: the write then a 256 MiB read of another "
                                           "buffer"}},
        "e2e": {"value": e2e_value, "unit": "DOF/s", "h2d_bytes_per_step": 8 * p.n,
                "d2h_bytes_per_step": 8 * p.n, "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "configs": extras,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="airg", choices=["airg", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the C2 / C3 secondary lines")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"],
                    help="solve arithmetic: fast (lane groups, FMA, fused level operators; within the parity "
                         "tolerance) or exact (the reference's bits)")
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
