"""Run reports in the reference's schema (reports.hpp / reports.cpp:18-133).

The reference CLI writes `stats.json` (hierarchy_report + solve_report) and
appends rows to `runs.csv`; the same documents from a GPU hierarchy let the
reference's tooling consume GPU runs unchanged. Field names,
nesting, the CSV column order and the printf formats follow reports.cpp;
tests/test_gpu_reports.py checks them against the reference's own output.
"""
from __future__ import annotations

import math
import os

from . import airg


def _max_theta(h: "airg.Hierarchy") -> float:
    """max_theta (reports.cpp:98-103): the largest post-DDC dominance ratio."""
    worst = 0.0
    for l in range(h.n_levels):
        worst = max(worst, h.level(l).max_theta_post)
    return worst


def hierarchy_report(h: "airg.Hierarchy") -> dict:
    """hierarchy_report (reports.cpp:18-51)."""
    levels = []
    for l in range(h.n_levels):
        lv = h.level(l)
        levels.append({
            "level": l, "n": lv.n, "nnz": lv.nnz, "n_f": lv.n_f, "n_c": lv.n_c,
            "max_theta_pre": lv.max_theta_pre, "max_theta_post": lv.max_theta_post,
            "ddc_alpha_diag": lv.alpha_diag, "ddc_converted": lv.ddc_converted,
            # A_ff keeps A's full diagonal, so it is structurally diagonal
            # exactly when it has one entry per row
            "aff_diagonal": lv.nnz_ff == lv.n_f,
            "nnz_r": lv.nnz_r, "nnz_p": lv.nnz_p, "nnz_aff_inv": lv.nnz_ffinv,
            "smoother_growth": lv.smoother_growth, "poly_attempts": lv.poly_attempts,
        })
    info = h.info()
    return {
        "levels": levels,
        "coarse": {"n": info.coarse_n, "nnz": info.coarse_nnz, "poly_order": h.coarse_poly_order,
                   "iterations": h.coarse_iterations, "solver_growth": info.coarse_growth},
        "level_count": h.n_levels + 1,
        "grid_complexity": info.grid_complexity,
        "operator_complexity": info.operator_complexity,
        "storage_complexity": info.storage_complexity,
        "max_theta": _max_theta(h),
    }


def solve_report(res: "airg.SolveResult") -> dict:
    """solve_report (reports.cpp:53-73); wall-clock numbers under "timing"."""
    st = res.stats
    return {
        "iterations": st.iterations, "converged": bool(st.converged),
        "residual_history": [float(r) for r in res.residual_history],
        "final_relative_residual": st.final_relative_residual,
        "flops": st.flops, "shadow_flops": st.shadow_flops, "work_units": st.work_units,
        "grid_complexity": st.grid_complexity, "operator_complexity": st.operator_complexity,
        "storage_complexity": st.storage_complexity,
        "timing": {"solve_seconds": st.solve_seconds, "wu_ratio": st.wu_ratio,
                   "c_grind_ns": st.c_grind_ns, "d_grind_ns": st.d_grind_ns},
    }


def partition_report(d: "airg.Dist", initial_ranks: int, threshold: float) -> dict:
    """partition_report (reports.cpp:75-101) for the row-slab distribution the
    GPU actually runs: the reference's replay rule (partition_model.cpp:77-112)
    on every hierarchy level, then the coarsest grid gathered on one GPU (the
    reference's model applies the rule once more there; the GPU gathers)."""
    levels, triggers = [], []
    for l in range(d.n_levels):
        li = d.level_info(l)
        n, nnz = d._levels[l]
        finite = math.isfinite(li["ratio_after"])
        levels.append({
            "level": l, "n": n, "nnz": nnz, "active_ranks": li["active"],
            "triggered": li["triggered"],
            "ratio": li["ratio_after"] if finite else None,
            "ratio_before_trigger": li["ratio_before"] if math.isfinite(li["ratio_before"]) else None,
            "local_share": li["share_after"] if math.isfinite(li["share_after"]) else 1.0,
        })
        if li["triggered"]:
            triggers.append(l)
    cn, cz = d._coarse
    levels.append({"level": d.n_levels, "n": cn, "nnz": cz, "active_ranks": 1,
                   "triggered": False, "ratio": None, "ratio_before_trigger": None, "local_share": 1.0,
                   "gathered": True})
    return {"initial_ranks": initial_ranks, "threshold": threshold, "levels": levels,
            "trigger_levels": triggers}


def csv_header() -> str:
    """csv_header (reports.cpp:105-109)."""
    return ("alpha,cf,levels,grid_complexity,operator_complexity,"
            "storage_complexity,iterations,work_units,max_theta,n,nnz,"
            "converged,final_relres,seed")


def csv_row(h: "airg.Hierarchy", stats, alpha: float, cf_name: str, seed: int) -> str:
    """csv_row (reports.cpp:111-126): same columns and printf formats."""
    info = h.info()
    top = h.level(0) if h.n_levels else None
    n = top.n if top else info.coarse_n
    nnz = top.nnz if top else info.coarse_nnz
    return ("%.6g,%s,%d,%.6g,%.6g,%.6g,%d,%.6g,%.6g,%d,%d,%d,%.6g,%d" % (
        alpha, cf_name, h.n_levels + 1, info.grid_complexity, info.operator_complexity,
        info.storage_complexity, stats.iterations, stats.work_units, _max_theta(h), n, nnz,
        1 if stats.converged else 0, stats.final_relative_residual, seed & (2**64 - 1)))


def append_csv(path, row: str) -> None:
    """append_csv (reports.cpp:128-133): header first when the file is new."""
    fresh = not os.path.exists(path)
    with open(path, "a") as f:
        if fresh:
            f.write(csv_header() + "\n")
        f.write(row + "\n")
