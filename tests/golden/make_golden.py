"""Generate tests/golden/*.npz from the REFERENCE build (oracle/_ref).

Run here, where /root/reference exists:   python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/airg_oracle.c) and, through it,
the GPU path, on machines without /root/reference. Each fixture stores the
problem (so the test does not depend on the generator), the reference's
level-0 CF split, every level's summary and polynomial coefficients, one
V-cycle and the Richardson solve.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import refpy  # noqa: E402
from paper_2408_08262_b200 import problems  # noqa: E402

# (name, builder, setup params)
CASES = [
    ("c0_full", lambda: problems.c0_structured_2d(128), problems.setup_params(0)),
    ("c1_64", lambda: problems.c1_unstructured_2d(64), problems.setup_params(1)),
    ("c2_16", lambda: problems.c2_structured_3d(16), dict(problems.setup_params(2), coarse_size_target=300)),
    ("c3_16x4", lambda: problems.c3_sn_2d(16, n_angles=4), dict(problems.setup_params(3), coarse_size_target=300)),
    ("c4_8", lambda: problems.c4_tets_3d(8, 8, 8), dict(problems.setup_params(4), coarse_size_target=300)),
]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def desk_problem(lib, nx, seed, jitter):
    import ctypes as C
    a = C.c_void_p()
    n = C.c_int64()
    b = np.zeros(200000)
    lib.call("desk_problem", nx, seed, jitter, C.byref(a), b, len(b), C.byref(n))
    m = refpy.Mat(lib, a, owned=True)
    return m, b[: n.value].copy()


def make_case(lib, name, p_rp, p_ci, p_v, b, prm):
    n = len(p_rp) - 1
    A = lib.mat(n, n, p_rp, p_ci, p_v)
    lab, pre, rep = refpy.cf_split(lib, A, prm, prm.get("seed", 0))
    h = refpy.setup(lib, A, **prm)
    info = h.info()
    nl = info.n_levels
    lv_n, lv_nnz, lv_nf, lv_eff, lv_coef, lv_conv = [], [], [], [], [], []
    lv_digest = []
    for l in range(nl):
        L = h.level(l)
        lv_n.append(L.n)
        lv_nnz.append(L.nnz)
        lv_nf.append(L.n_f)
        lv_eff.append(L.effective_order)
        lv_conv.append(L.ddc_converted)
        lv_coef.append(np.array(L.coefficients[: prm["poly_order"] + 1]))
        lv_digest.append(digest(h.labels(l)) + ":" + "|".join(
            digest(np.concatenate([x.view(np.uint8) for x in h.matrix(l, w).arrays()])) for w in range(7)))
    scfg = refpy.abi.solve_config(coarse_iterations=prm.get("coarse_iterations", 3))
    xv = h.vcycle(b, scfg)
    x, st, hist = h.solve(b, scfg)
    out = dict(
        rp=p_rp, ci=p_ci, v=p_v, b=b,
        params=np.array([repr(prm)]),
        labels=lab, labels_pre=pre,
        cf_report=np.array([rep.n_f_pre, rep.n_f, rep.n_c, rep.n_converted, rep.s_nnz], np.int64),
        cf_theta=np.array([rep.max_theta, rep.alpha_diag]),
        n_levels=np.array(nl), coarse_n=np.array(info.coarse_n),
        coarse_coeffs=np.array(info.coarse_coefficients[: prm["coarse_poly_order"] + 1]),
        coarse_eff=np.array(info.coarse_effective_order),
        level_n=np.array(lv_n), level_nnz=np.array(lv_nnz), level_nf=np.array(lv_nf),
        level_eff=np.array(lv_eff), level_conv=np.array(lv_conv),
        level_coeffs=np.array(lv_coef) if nl else np.zeros((0, prm["poly_order"] + 1)),
        level_digest=np.array(lv_digest),
        complexities=np.array([info.grid_complexity, info.operator_complexity, info.storage_complexity]),
        vcycle=xv, x=x, history=hist,
        solve=np.array([st.iterations, st.converged, st.flops], np.int64),
        final_rel=np.array(st.final_relative_residual),
    )
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: n={n} levels={nl} its={st.iterations} rel={st.final_relative_residual:.3e}")


def main():
    lib = refpy.ref()
    if lib is None:
        raise SystemExit("oracle/_ref unavailable: run where /root/reference exists")
    for name, builder, prm in CASES:
        p = builder()
        make_case(lib, name, p.row_offsets, p.cols, p.vals, p.b, prm)
    # the reference's own desk operator (transport.cpp, SUPG 4-angle) with the
    # serial settings of test_solve.cpp:129-150
    A, b = desk_problem(lib, 15, 1, 0.3)
    rp, ci, v = A.arrays()
    prm = dict(strength_alpha=0.5, poly_order=3, sparsity_order=1, coarse_poly_order=3,
               coarse_iterations=1, drop_coarse=0.0075, drop_restrict=0.025, coarse_size_target=0,
               seed=7)
    make_case(lib, "desk15", rp, ci, v, b, prm)


if __name__ == "__main__":
    main()
