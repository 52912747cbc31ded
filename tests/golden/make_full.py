"""Full-size parity fixtures (SURVEY §8c P1/P2/P5 at the BASELINE sizes),
generated from the REFERENCE build (oracle/_ref) -- TEST INFRASTRUCTURE.

Run here, where /root/reference exists:
    python tests/golden/make_full.py 1 2 3 4        (about 20 min serial)

The GPU box has no /root/reference and the reference's serial setup of the
8.4 M-unknown C3 system takes minutes, so the fixtures carry what the
full-size parity tests compare, not the problem (the test regenerates it
with problems.make and checks `problem_digest` first):
  * every level's summary: n, nnz, n_f, n_c, DDC conversions, effective
    order, coefficients, smoother growth, attempts, and the sha256 of the
    labels and of the seven level matrices (A, A_ff, A_fc, A_cf, Aff^-1, R, P);
  * the coarse grid's summary;
  * the solve: Richardson (solve.cpp:167-259) where it converges, and the
    outer GMRES(30) around the reference's own vcycle() (oracle/ref_capi.cpp
    `ref_gmres`) for C0 and for C4, where the reference's Richardson
    diverges (residual x5.4 per iteration from iteration 4; see
    `c4_richardson_history`); iterations, final residual, history, the
    sha256 of x and x at 65,536 seeded indices (relative-L2 estimate; the
    exact comparison goes through the injection-mode solve, whose x must
    hash identically);
  * the reference's serial timings on this container (setup, solve).
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import refpy  # noqa: E402
from paper_2408_08262_b200 import problems  # noqa: E402

OUT = os.path.join(HERE, "full")
N_SAMPLE = 65536
GMRES_CONFIGS = (0, 4)  # outer GMRES(30): C0 names it; C4's Richardson diverges


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem_digest(p) -> str:
    h = hashlib.sha256()
    for a in (np.asarray(p.row_offsets, np.int64), np.asarray(p.cols, np.int64),
              np.asarray(p.vals, np.float64), np.asarray(p.b, np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sample_index(n: int) -> np.ndarray:
    """65,536 distinct seeded indices (sorted) -- the same on every machine."""
    rs = np.random.Generator(np.random.PCG64(20240826))
    k = min(n, N_SAMPLE)
    return np.sort(rs.choice(n, size=k, replace=False)).astype(np.int64)


def matrix_digest(m) -> str:
    return digest(np.concatenate([x.view(np.uint8) for x in m.arrays()]))


def make(cfg: int) -> None:
    lib = refpy.ref()
    if lib is None:
        raise SystemExit("oracle/_ref unavailable: run where /root/reference exists")
    p = problems.make(cfg)
    prm = problems.setup_params(cfg)
    A = lib.mat_from_problem(p)
    lab, _, rep = refpy.cf_split(lib, A, prm, prm["seed"])
    t0 = time.perf_counter()
    h = refpy.setup(lib, A, **prm)
    setup_s = time.perf_counter() - t0
    info = h.info()
    nl = info.n_levels
    cols = {k: [] for k in ("n", "nnz", "nf", "nc", "conv", "eff", "growth", "attempts", "coef",
                            "lab_digest", "mat_digest", "nnz_ffinv", "nnz_r")}
    for l in range(nl):
        L = h.level(l)
        cols["n"].append(L.n)
        cols["nnz"].append(L.nnz)
        cols["nf"].append(L.n_f)
        cols["nc"].append(L.n_c)
        cols["conv"].append(L.ddc_converted)
        cols["eff"].append(L.effective_order)
        cols["growth"].append(L.smoother_growth)
        cols["attempts"].append(L.poly_attempts)
        cols["coef"].append(np.array(L.coefficients[: prm["poly_order"] + 1]))
        cols["nnz_ffinv"].append(L.nnz_ffinv)
        cols["nnz_r"].append(L.nnz_r)
        cols["lab_digest"].append(digest(h.labels(l)))
        cols["mat_digest"].append("|".join(matrix_digest(h.matrix(l, w)) for w in range(7)))
    outer = 1 if cfg in GMRES_CONFIGS else 0
    scfg = refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"], outer=outer,
                                  max_iterations=400)
    t0 = time.perf_counter()
    x, st, hist = h.solve(p.b, scfg, cap=4096)
    solve_s = time.perf_counter() - t0
    idx = sample_index(p.n)
    out = dict(
        config=np.array(cfg), n=np.array(p.n), nnz=np.array(p.nnz),
        problem_digest=np.array(problem_digest(p)), params=np.array([repr(prm)]),
        labels0_digest=np.array(digest(lab)),
        cf_report=np.array([rep.n_f_pre, rep.n_f, rep.n_c, rep.n_converted, rep.s_nnz], np.int64),
        cf_theta=np.array([rep.max_theta, rep.alpha_diag]),
        n_levels=np.array(nl), coarse_n=np.array(info.coarse_n), coarse_nnz=np.array(info.coarse_nnz),
        coarse_coeffs=np.array(info.coarse_coefficients[: prm["coarse_poly_order"] + 1]),
        coarse_eff=np.array(info.coarse_effective_order), coarse_growth=np.array(info.coarse_growth),
        coarse_attempts=np.array(info.coarse_attempts),
        level_n=np.array(cols["n"], np.int64), level_nnz=np.array(cols["nnz"], np.int64),
        level_nf=np.array(cols["nf"], np.int64), level_nc=np.array(cols["nc"], np.int64),
        level_conv=np.array(cols["conv"], np.int64), level_eff=np.array(cols["eff"], np.int64),
        level_growth=np.array(cols["growth"]), level_attempts=np.array(cols["attempts"], np.int64),
        level_nnz_ffinv=np.array(cols["nnz_ffinv"], np.int64), level_nnz_r=np.array(cols["nnz_r"], np.int64),
        level_coeffs=np.array(cols["coef"]), level_labels_digest=np.array(cols["lab_digest"]),
        level_matrix_digest=np.array(cols["mat_digest"]),
        complexities=np.array([info.grid_complexity, info.operator_complexity, info.storage_complexity]),
        outer=np.array(outer),
        solve=np.array([st.iterations, st.converged], np.int64), final_rel=np.array(st.final_relative_residual),
        history=hist, x_digest=np.array(digest(x)), x_norm=np.array(np.linalg.norm(x)),
        x_index=idx, x_sample=x[idx],
        ref_setup_s=np.array(setup_s), ref_solve_s=np.array(solve_s),
    )
    if cfg == 4:  # the reference's own Richardson on the same hierarchy (diverges)
        r_cfg = refpy.abi.solve_config(coarse_iterations=prm["coarse_iterations"], max_iterations=12)
        _, rst, rhist = h.solve(p.b, r_cfg, cap=64)
        out["c4_richardson_history"] = rhist
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"c{cfg}.npz"), **out)
    print(f"c{cfg}: n={p.n} levels={nl} outer={outer} its={st.iterations} rel={st.final_relative_residual:.3e} "
          f"setup {setup_s:.1f} s solve {solve_s:.1f} s", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["1", "2", "3", "4"]:
        make(int(a))
