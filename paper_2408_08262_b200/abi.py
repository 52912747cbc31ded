"""ctypes mirrors of the plain-C structs in include/airg_c.h.

Shared by the product binding (airg.py) and the test-only oracle bindings;
field order and types must match the header exactly.
"""
from __future__ import annotations

import ctypes as C


class SetupConfig(C.Structure):
    """airg_setup_config == airgraph::SetupConfig (air.hpp:16-43)."""
    _fields_ = [
        ("strength_alpha", C.c_double),
        ("cf", C.c_int32),
        ("ddc_enabled", C.c_int32),
        ("ddc_fraction", C.c_double),
        ("ddc_bins", C.c_int64),
        ("max_loops", C.c_int64),
        ("poly_order", C.c_int64),
        ("sparsity_order", C.c_int64),
        ("drop_coarse", C.c_double),
        ("drop_restrict", C.c_double),
        ("coarse_size_target", C.c_int64),
        ("coarse_poly_order", C.c_int64),
        ("coarse_iterations", C.c_int64),
        ("max_levels", C.c_int64),
        ("prolongation", C.c_int32),
        ("weight_mode", C.c_int32),
        ("seed", C.c_uint64),
        ("fused_smooths", C.c_int32),
        ("_pad", C.c_int32),
    ]


class SolveConfig(C.Structure):
    """airg_solve_config == airgraph::SolveConfig (solve.hpp:11-19) + outer."""
    _fields_ = [
        ("rtol", C.c_double),
        ("max_iterations", C.c_int64),
        ("up_f_smooths", C.c_int64),
        ("down_smooths", C.c_int64),
        ("coarse_iterations", C.c_int64),
        ("collect_timing", C.c_int32),
        ("outer", C.c_int32),
        ("nddofs", C.c_int64),
        ("gmres_restart", C.c_int64),
        ("fast", C.c_int32),
        ("_pad2", C.c_int32),
    ]


class SolveStats(C.Structure):
    """airg_solve_stats == airgraph::SolveStats (solve.hpp:21-39)."""
    _fields_ = [
        ("iterations", C.c_int64),
        ("converged", C.c_int32),
        ("_pad", C.c_int32),
        ("final_relative_residual", C.c_double),
        ("flops", C.c_uint64),
        ("shadow_flops", C.c_uint64),
        ("work_units", C.c_double),
        ("grid_complexity", C.c_double),
        ("operator_complexity", C.c_double),
        ("storage_complexity", C.c_double),
        ("solve_seconds", C.c_double),
        ("wu_ratio", C.c_double),
        ("c_grind_ns", C.c_double),
        ("d_grind_ns", C.c_double),
        ("history_len", C.c_int64),
    ]


class LevelInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nnz", C.c_int64),
        ("n_f", C.c_int64), ("n_c", C.c_int64),
        ("n_f_pre", C.c_int64), ("ddc_converted", C.c_int64),
        ("nnz_ff", C.c_int64), ("nnz_fc", C.c_int64), ("nnz_cf", C.c_int64),
        ("nnz_ffinv", C.c_int64), ("nnz_r", C.c_int64), ("nnz_p", C.c_int64),
        ("max_theta_pre", C.c_double), ("alpha_diag", C.c_double),
        ("max_theta_post", C.c_double), ("smoother_growth", C.c_double),
        ("poly_attempts", C.c_int64), ("effective_order", C.c_int64),
        ("coefficients", C.c_double * 32),
    ]


class HierInfo(C.Structure):
    _fields_ = [
        ("n_levels", C.c_int64),
        ("coarse_n", C.c_int64), ("coarse_nnz", C.c_int64), ("coarse_inv_nnz", C.c_int64),
        ("coarse_effective_order", C.c_int64), ("coarse_attempts", C.c_int64),
        ("coarse_growth", C.c_double),
        ("coarse_coefficients", C.c_double * 32),
        ("grid_complexity", C.c_double), ("operator_complexity", C.c_double),
        ("storage_complexity", C.c_double),
    ]


class CfReport(C.Structure):
    _fields_ = [
        ("n_f_pre", C.c_int64), ("n_f", C.c_int64), ("n_c", C.c_int64),
        ("n_converted", C.c_int64),
        ("max_theta", C.c_double), ("alpha_diag", C.c_double),
        ("s_nnz", C.c_int64),
    ]


class Injection(C.Structure):
    _fields_ = [
        ("n_levels", C.c_int64),
        ("stride", C.c_int64),
        ("level_coeffs", C.POINTER(C.c_double)),
        ("level_eff_order", C.POINTER(C.c_int64)),
        ("coarse_coeffs", C.POINTER(C.c_double)),
        ("coarse_eff_order", C.c_int64),
    ]


SETUP_DEFAULTS = dict(
    strength_alpha=0.5, cf=0, ddc_enabled=1, ddc_fraction=0.10, ddc_bins=1000,
    max_loops=3, poly_order=6, sparsity_order=1, drop_coarse=0.001,
    drop_restrict=0.01, coarse_size_target=3000, coarse_poly_order=12,
    coarse_iterations=3, max_levels=0, prolongation=0, weight_mode=0, seed=0, fused_smooths=-1, _pad=0)

SOLVE_DEFAULTS = dict(
    rtol=1e-10, max_iterations=200, up_f_smooths=2, down_smooths=0,
    coarse_iterations=3, collect_timing=1, outer=0, nddofs=0, gmres_restart=30, fast=0, _pad2=0)


def setup_config(**kw) -> SetupConfig:
    d = dict(SETUP_DEFAULTS)
    for k, v in kw.items():
        if k not in d:
            raise KeyError(f"unknown setup parameter {k}")
        d[k] = v
    return SetupConfig(**d)


def solve_config(**kw) -> SolveConfig:
    d = dict(SOLVE_DEFAULTS)
    for k, v in kw.items():
        if k not in d:
            raise KeyError(f"unknown solve parameter {k}")
        d[k] = v
    return SolveConfig(**d)
