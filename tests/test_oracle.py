"""Pin the C restatement oracle (oracle/airg_oracle.c):
  * against the committed golden fixtures generated from the REFERENCE build
    (tests/golden/make_golden.py) -- runs everywhere;
  * against the reference build itself (oracle/_ref) when it is present.
Everything must be bit-identical: labels, every level matrix, the
polynomial coefficients, one V-cycle, the solution and residual history.
"""
import glob
import hashlib
import os

import numpy as np
import pytest

import refpy
from backends import random_sparse, same_bits
from paper_2408_08262_b200 import abi

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _params(g):
    return eval(str(g["params"][0]))  # repr(dict) written by make_golden.py


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_port_matches_reference_golden(port, path):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    A = port.mat(n, n, g["rp"], g["ci"], g["v"])
    lab, pre, rep = refpy.cf_split(port, A, prm, prm.get("seed", 0))
    assert np.array_equal(lab, g["labels"]) and np.array_equal(pre, g["labels_pre"])
    assert [rep.n_f_pre, rep.n_f, rep.n_c, rep.n_converted, rep.s_nnz] == list(g["cf_report"])
    assert same_bits([rep.max_theta, rep.alpha_diag], g["cf_theta"])
    h = refpy.setup(port, A, **prm)
    info = h.info()
    assert info.n_levels == int(g["n_levels"]) and info.coarse_n == int(g["coarse_n"])
    for l in range(info.n_levels):
        L = h.level(l)
        assert (L.n, L.nnz, L.n_f, L.effective_order, L.ddc_converted) == (
            g["level_n"][l], g["level_nnz"][l], g["level_nf"][l], g["level_eff"][l], g["level_conv"][l])
        assert same_bits(np.array(L.coefficients[: prm["poly_order"] + 1]), g["level_coeffs"][l])
        dig = _digest(h.labels(l)) + ":" + "|".join(
            _digest(np.concatenate([x.view(np.uint8) for x in h.matrix(l, w).arrays()])) for w in range(7))
        assert dig == str(g["level_digest"][l]), f"level {l} differs"
    assert same_bits(np.array(info.coarse_coefficients[: prm["coarse_poly_order"] + 1]), g["coarse_coeffs"])
    scfg = refpy.abi.solve_config(coarse_iterations=prm.get("coarse_iterations", 3))
    assert same_bits(h.vcycle(g["b"], scfg), g["vcycle"])
    x, st, hist = h.solve(g["b"], scfg)
    assert [st.iterations, st.converged, st.flops] == list(g["solve"])
    assert same_bits(x, g["x"]) and same_bits(hist, g["history"])


def test_desk_reference_bands(port):
    """test_solve.cpp:129-185 bands on the reference's own desk operator
    (<= 18 iterations, <= 100 WUs, monotone within 2 slips)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "desk15.npz"))
    prm = _params(g)
    n = len(g["rp"]) - 1
    A = port.mat(n, n, g["rp"], g["ci"], g["v"])
    h = refpy.setup(port, A, **prm)
    x, st, hist = h.solve(g["b"], refpy.abi.solve_config(coarse_iterations=1))
    assert st.converged and st.iterations <= 18 and st.work_units <= 100.0
    assert sum(hist[k] >= hist[k - 1] for k in range(1, len(hist))) <= 2
    assert -np.log10(st.final_relative_residual) / st.iterations >= 0.5


def test_zero_rhs_converges_immediately(port):  # test_solve.cpp:171-181
    a = random_sparse(10, 0.4, 6)
    A = port.mat(*a)
    h = refpy.setup(port, A, coarse_size_target=100)
    x, st, hist = h.solve(np.zeros(10))
    assert st.converged and st.iterations == 0


def test_nonconvergence_reported(port):  # test_solve.cpp:187-201
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "desk15.npz"))
    prm = _params(g)
    n = len(g["rp"]) - 1
    h = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    x, st, hist = h.solve(g["b"], refpy.abi.solve_config(max_iterations=1, coarse_iterations=1))
    assert not st.converged and st.iterations == 1 and st.final_relative_residual > 1e-10


def test_setup_stall_raises(port):  # test_air.cpp:280-291 (PMIS baseline stalls on I)
    A = port.mat(50, 50, np.arange(51), np.arange(50), np.ones(50))
    with pytest.raises(RuntimeError, match="stall"):
        refpy.setup(port, A, cf=1, ddc_enabled=0, coarse_size_target=5, poly_order=2)


def test_gmres_oracle_converges(port):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c0_full.npz"))
    prm = _params(g)
    n = len(g["rp"]) - 1
    h = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    x, st, hist = h.solve(g["b"], refpy.abi.solve_config(outer=1, coarse_iterations=3))
    assert st.converged and st.final_relative_residual <= 1e-10
    xr, sr, _ = h.solve(g["b"], refpy.abi.solve_config(coarse_iterations=3))
    assert st.iterations <= sr.iterations
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-8


# ---- directly against the reference build (only where /root/reference exists)
@pytest.mark.parametrize("seed", range(4))
def test_port_components_match_reference(port, reflib, seed):
    a = random_sparse(40, 0.12, 1000 + seed)
    A, R = port.mat(*a), reflib.mat(*a)
    b = random_sparse(40, 0.12, 2000 + seed)
    B, RB = port.mat(*b), reflib.mat(*b)
    for op, args in [("spgemm", ()), ("drop", (0.3, 1)), ("drop", (0.3, 0))]:
        if op == "spgemm":
            x = refpy.binop(port, op, A.h, B.h).arrays()
            y = refpy.binop(reflib, op, R.h, RB.h).arrays()
        else:
            x = refpy.binop(port, op, A.h, *args).arrays()
            y = refpy.binop(reflib, op, R.h, *args).arrays()
        assert all(same_bits(u.astype(np.float64) if u.dtype != np.float64 else u,
                             v.astype(np.float64) if v.dtype != np.float64 else v) for u, v in zip(x, y))
    for m in (2, 5, 9):
        c1 = np.zeros(m)
        c2 = np.zeros(m)
        import ctypes as C
        e1, e2 = C.c_int64(), C.c_int64()
        port.call("poly_coefficients", A.h, m, seed, c1, C.byref(e1))
        reflib.call("poly_coefficients", R.h, m, seed, c2, C.byref(e2))
        assert same_bits(c1, c2) and e1.value == e2.value


def test_port_setup_matches_reference_c2_small(port, reflib):
    from paper_2408_08262_b200 import problems
    p = problems.c2_structured_3d(20)
    prm = dict(problems.setup_params(2), coarse_size_target=500)
    h1 = refpy.setup(port, port.mat_from_problem(p), **prm)
    h2 = refpy.setup(reflib, reflib.mat_from_problem(p), **prm)
    assert h1.info().n_levels == h2.info().n_levels
    for l in range(h1.info().n_levels):
        for w in range(7):
            for u, v in zip(h1.matrix(l, w).arrays(), h2.matrix(l, w).arrays()):
                assert np.array_equal(u.view(np.uint8), v.view(np.uint8))
    s1 = h1.solve(p.b, refpy.abi.solve_config())
    s2 = h2.solve(p.b, refpy.abi.solve_config())
    assert same_bits(s1[0], s2[0]) and same_bits(s1[2], s2[2])


def _same_mat(x, y):
    (a, b, c), (d, e, f) = x.arrays(), y.arrays()
    return x.dims() == y.dims() and np.array_equal(a, d) and np.array_equal(b, e) and same_bits(c, f)


@pytest.mark.parametrize("seed", [1, 2])
def test_port_single_ops_match_reference(port, reflib, seed):
    """dominance_report, build_label_map, build_restriction /
    build_prolongation / coarse_matrix, apply_polynomial and f_smooth of the
    C restatement against the reference build, bit for bit."""
    import ctypes as C
    a = random_sparse(80, 0.08, 300 + seed)
    A, R = port.mat(*a), reflib.mat(*a)
    lab = np.zeros(80, np.uint8)
    rep = abi.CfReport()
    port.call("cf_split", A.h, 0.5, 3, seed, 0, 1, 0.1, 1000, lab, None, C.byref(rep))
    lm_p, lm_r = refpy.build_label_map(port, lab), refpy.build_label_map(reflib, lab)
    assert all(np.array_equal(u, v) for u, v in zip(lm_p, lm_r))
    blocks = []
    for lib, M in ((port, A), (reflib, R)):
        o = [C.c_void_p(), C.c_void_p(), C.c_void_p()]
        lib.call("extract_blocks", M.h, lab, *[C.byref(x) for x in o])
        blocks.append([refpy.Mat(lib, x, True) for x in o])
    (pff, pfc, pcf), (rff, rfc, rcf) = blocks
    for bins in (1, 9, 1000):
        x, y = refpy.dominance_report(port, pff, bins), refpy.dominance_report(reflib, rff, bins)
        assert same_bits(x[0], y[0]) and np.array_equal(x[1], y[1]) and x[2] == y[2]
    co = np.zeros(4)
    eff = C.c_int64()
    reflib.call("poly_coefficients", rff.h, 4, seed, co, C.byref(eff))
    qp = refpy.binop(port, "poly_assemble", pff.h, co, 4, eff.value, 1)
    qr = refpy.binop(reflib, "poly_assemble", rff.h, co, 4, eff.value, 1)
    rp_ = refpy.binop(port, "build_restriction", pcf.h, qp.h, 0.01, lab, 80)
    rr_ = refpy.binop(reflib, "build_restriction", rcf.h, qr.h, 0.01, lab, 80)
    assert _same_mat(rp_, rr_)
    sp, sr = C.c_void_p(), C.c_void_p()
    port.call("strength", A.h, 0.5, C.byref(sp), None)
    reflib.call("strength", R.h, 0.5, C.byref(sr), None)
    SP, SR = refpy.Mat(port, sp, True), refpy.Mat(reflib, sr, True)
    pp = refpy.binop(port, "build_prolongation", A.h, SP.h, lab)
    pr = refpy.binop(reflib, "build_prolongation", R.h, SR.h, lab)
    assert _same_mat(pp, pr)
    cp = refpy.binop(port, "coarse_matrix", rp_.h, A.h, pp.h, 0.001)
    cr = refpy.binop(reflib, "coarse_matrix", rr_.h, R.h, pr.h, 0.001)
    assert _same_mat(cp, cr)
    b = np.random.default_rng(seed).random(80)
    assert same_bits(refpy.apply_polynomial(port, A, co, eff.value, b),
                     refpy.apply_polynomial(reflib, R, co, eff.value, b))
    from paper_2408_08262_b200 import problems
    pb = problems.c2_structured_3d(10)
    prm = dict(problems.setup_params(2), coarse_size_target=150)
    hp = refpy.setup(port, port.mat_from_problem(pb), **prm)
    hr = refpy.setup(reflib, reflib.mat_from_problem(pb), **prm)
    x0 = np.random.default_rng(seed + 7).random(pb.n)
    assert same_bits(hp.f_smooth(0, pb.b, x0), hr.f_smooth(0, pb.b, x0))
