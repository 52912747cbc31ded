"""GPU parity against the CPU oracle through the C-ABI.

P1  level-0 CF labels bit-exact (all five configs);
P2  the GPU CF split of every oracle level operator bit-exact;
P3/P4 coefficient-injection hierarchy bit-identical (every level matrix),
    one V-cycle bit-identical, Richardson iterates bit-identical;
P5  native mode: final relative residual <= 1e-10 (fresh matvec),
    iterations within +-1, solution within 1e-8 relative L2.
"""
import glob
import hashlib
import os

import numpy as np
import pytest

import refpy
from backends import same_bits
from paper_2408_08262_b200 import airg, problems

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
TOL_X = 1e-8     # north_star: solution within 1e-8 relative L2
TOL_RES = 1e-10  # north_star: final relative residual <= 1e-10


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _params(g):
    return eval(str(g["params"][0]))


def _sm(p):
    return airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)


def _injection(oh, prm):
    info = oh.info()
    return {"levels": [(list(oh.level(l).coefficients[: prm["poly_order"] + 1]), oh.level(l).effective_order)
                       for l in range(info.n_levels)],
            "coarse": (list(info.coarse_coefficients[: prm["coarse_poly_order"] + 1]),
                       info.coarse_effective_order)}


CF_CASES = [(0, 1.0), (1, 0.25), (2, 0.25), (3, 0.125), (4, 0.25), (1, 1.0), (2, 1.0), (3, 1.0), (4, 1.0)]


@pytest.mark.parametrize("cfg,scale", CF_CASES, ids=[f"C{c}x{s}" for c, s in CF_CASES])
def test_p1_level0_cf_labels_bit_exact(port, cfg, scale):
    p = problems.make(cfg, scale)
    prm = problems.setup_params(cfg)
    seed = int(problems.mix(np.uint64(0), np.uint64(0)))  # level_seed of level 0 (air.cpp:324)
    lab, pre, rep = airg.cf_split(_sm(p), prm["strength_alpha"], prm["max_loops"], seed)
    ol, op, orep = refpy.cf_split(port, port.mat_from_problem(p), prm, seed)
    assert np.array_equal(pre, op), "PMISR labels differ"
    assert np.array_equal(lab, ol), "post-DDC labels differ"
    assert (rep.n_f_pre, rep.n_converted, rep.s_nnz) == (orep.n_f_pre, orep.n_converted, orep.s_nnz)
    assert same_bits([rep.max_theta, rep.alpha_diag], [orep.max_theta, orep.alpha_diag])
    # ... and at 2/4/8 GPUs (row slabs, emulated ranks)
    for P in (2, 4, 8):
        dl, drep = airg.dist_cf_split(_sm(p), P, alpha=prm["strength_alpha"], max_loops=prm["max_loops"],
                                      seed=seed)
        assert np.array_equal(dl, ol), f"{P}-slab labels differ"
        assert drep.n_converted == orep.n_converted
    # size-independent property: F independent in S u S^T
    s = airg.strength(_sm(p), prm["strength_alpha"])
    d = np.repeat(np.arange(p.n), np.diff(s.row_offsets))
    assert not ((pre[d] == 0) & (pre[s.col_indices] == 0)).any()


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_p2_every_level_cf_split(port, path):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    oh = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    mats, seeds, reps = [], [], []
    for l in range(oh.info().n_levels):
        rp, ci, v = oh.matrix(l, 0).arrays()
        a = airg.SparseMatrix.from_arrays(len(rp) - 1, len(rp) - 1, rp, ci, v)
        seed = int(problems.mix(np.uint64(prm.get("seed", 0)), np.uint64(l)))
        lab, _, rep = airg.cf_split(a, prm["strength_alpha"], prm.get("max_loops", 3), seed,
                                    ddc_fraction=prm.get("ddc_fraction", 0.1))
        assert np.array_equal(lab, oh.labels(l)), f"level {l}"
        mats.append(airg.DeviceCSR.upload(a))
        seeds.append(seed)
        reps.append(rep)
    # every level in one batched call (one synchronisation): same labels and reports
    bl, br = airg.cf_split_batch_device(mats, seeds, prm["strength_alpha"], prm.get("max_loops", 3),
                                        ddc_fraction=prm.get("ddc_fraction", 0.1))
    for l, (t, r) in enumerate(zip(bl, br)):
        assert np.array_equal(t.cpu().numpy()[: len(oh.labels(l))], oh.labels(l)), f"batched level {l}"
        assert (r.n_f, r.n_f_pre, r.n_converted, r.s_nnz) == \
            (reps[l].n_f, reps[l].n_f_pre, reps[l].n_converted, reps[l].s_nnz)
        assert same_bits([r.max_theta, r.alpha_diag], [reps[l].max_theta, reps[l].alpha_diag])


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_p4_injected_hierarchy_bit_identical(port, path):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    oh = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
    h = airg.setup(a, injection=_injection(oh, prm), **prm)
    assert h.n_levels == oh.info().n_levels == int(g["n_levels"])
    for l in range(h.n_levels):
        assert np.array_equal(h.labels(l), oh.labels(l))
        for w in range(7):
            got = h.matrix(l, w)
            exp = oh.matrix(l, w).arrays()
            assert np.array_equal(got.row_offsets, exp[0]), (l, w)
            assert np.array_equal(got.col_indices, exp[1]), (l, w)
            assert same_bits(got.values, exp[2]), (l, w)
        L, OL = h.level(l), oh.level(l)
        assert (L.n_f_pre, L.ddc_converted) == (OL.n_f_pre, OL.ddc_converted)
        assert same_bits([L.max_theta_pre, L.alpha_diag, L.max_theta_post],
                         [OL.max_theta_pre, OL.alpha_diag, OL.max_theta_post])
    for w in (0, 4):
        got = h.matrix(h.n_levels, w)
        exp = oh.matrix(h.n_levels, w).arrays()
        assert np.array_equal(got.col_indices, exp[1]) and same_bits(got.values, exp[2])
    ci = prm.get("coarse_iterations", 3)
    xv = h.vcycle(g["b"], coarse_iterations=ci)
    assert same_bits(xv, g["vcycle"]), "V-cycle not bit-identical to the reference"
    res = airg.richardson_solve(h, g["b"], coarse_iterations=ci)
    assert res.stats.iterations == int(g["solve"][0])
    assert res.stats.flops == int(g["solve"][2])  # work units identical
    assert same_bits(res.x, g["x"]), "Richardson iterates differ"
    np.testing.assert_allclose(res.residual_history, g["history"], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("cf", [1, 2])
@pytest.mark.parametrize("path", GOLDEN[:4], ids=lambda p: os.path.basename(p)[:-4])
def test_pmis_baselines_injected_hierarchy(port, path, cf):
    """The paper's comparison splittings (cli.cpp:141-147: PMIS and PMIS-swap,
    DDC off): every level's labels and operators bit-identical to the oracle
    with injected coefficients, and the V-cycle too."""
    g = np.load(path)
    prm = dict(_params(g), cf=cf, ddc_enabled=0)
    n = len(g["rp"]) - 1
    try:
        oh = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    except RuntimeError as e:  # the baseline may stall; the GPU must stall the same way
        with pytest.raises(airg.AirgRuntimeError, match="stall"):
            airg.setup(airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]), **prm)
        return
    a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
    h = airg.setup(a, injection=_injection(oh, prm), **prm)
    assert h.n_levels == oh.info().n_levels
    for l in range(h.n_levels):
        assert np.array_equal(h.labels(l), oh.labels(l)), l
        for w in range(7):
            got = h.matrix(l, w)
            exp = oh.matrix(l, w).arrays()
            assert np.array_equal(got.col_indices, exp[1]) and same_bits(got.values, exp[2]), (l, w)
    ci = prm.get("coarse_iterations", 3)
    xo = oh.vcycle(g["b"], refpy.abi.solve_config(coarse_iterations=ci))
    assert same_bits(h.vcycle(g["b"], coarse_iterations=ci), xo)
    # the bare splitting through the C-ABI (DDC off: the level-0 labels)
    seed = int(problems.mix(np.uint64(prm.get("seed", 0)), np.uint64(0)))
    lab = airg.pmis(a, prm["strength_alpha"], swap=cf == 2, seed=seed)
    assert np.array_equal(lab, oh.labels(0))


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_p5_native_solve_within_tolerance(port, path):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
    h = airg.setup(a, **prm)
    ci = prm.get("coarse_iterations", 3)
    res = airg.richardson_solve(h, g["b"], coarse_iterations=ci)
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    assert abs(res.stats.iterations - int(g["solve"][0])) <= 1
    # fresh matvec residual on the host (the reference's own definition)
    r = g["b"] - airg.spmv(a, res.x)
    assert np.linalg.norm(r) / np.linalg.norm(g["b"]) <= TOL_RES
    assert np.linalg.norm(res.x - g["x"]) / np.linalg.norm(g["x"]) <= TOL_X
    # native coefficients track the reference's long-double fit
    oh = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    assert h.n_levels == oh.info().n_levels
    for l in range(h.n_levels):
        c1 = np.array(h.level(l).coefficients[: prm["poly_order"] + 1])
        c2 = np.array(oh.level(l).coefficients[: prm["poly_order"] + 1])
        assert h.level(l).effective_order == oh.level(l).effective_order, l
        assert np.abs(c1 - c2).max() <= 1e-7 * max(1.0, np.abs(c2).max()), l


@pytest.mark.parametrize("path", GOLDEN[:3], ids=lambda p: os.path.basename(p)[:-4])
def test_gmres_matches_oracle_gmres(port, path):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    oh = refpy.setup(port, port.mat(n, n, g["rp"], g["ci"], g["v"]), **prm)
    a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
    h = airg.setup(a, injection=_injection(oh, prm), **prm)
    ci = prm.get("coarse_iterations", 3)
    res = airg.gmres_solve(h, g["b"], coarse_iterations=ci)
    xo, so, _ = oh.solve(g["b"], refpy.abi.solve_config(outer=1, coarse_iterations=ci))
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    assert abs(res.stats.iterations - so.iterations) <= 1
    assert np.linalg.norm(res.x - xo) / np.linalg.norm(xo) <= TOL_X


def test_c2_full_native_solve(port):
    """BASELINE config 2 at full size: native GPU setup + Richardson against
    the oracle's hierarchy-independent tolerance contract."""
    p = problems.make(2)
    prm = problems.setup_params(2)
    a = _sm(p)
    h = airg.setup(a, **prm)
    res = airg.richardson_solve(h, p.b, coarse_iterations=prm["coarse_iterations"])
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    r = p.b - refpy.spmv(port, port.mat_from_problem(p), res.x)
    assert np.linalg.norm(r) / np.linalg.norm(p.b) <= TOL_RES * 1.01
    g = airg.gmres_solve(h, p.b, coarse_iterations=prm["coarse_iterations"])
    assert g.stats.converged and np.linalg.norm(g.x - res.x) / np.linalg.norm(res.x) <= 1e-8


@pytest.mark.parametrize("cfg", [0, 1, 3, 4])
def test_full_size_native_solves(cfg):
    """Every BASELINE config at full size: native setup + solve converges to
    rtol 1e-10, checked by a host scipy matvec independent of the GPU. C0
    and C4 use the outer GMRES: C0's config names it, and on C4 the level-0
    polynomial smoother misses the growth bound on every attempt (growth
    2.33 at full size, 1.04 at half size -- the compiled reference reports
    the same 1.0387 at half size) so plain Richardson stagnates there, in
    the reference as here."""
    import scipy.sparse as sp
    p = problems.make(cfg)
    prm = problems.setup_params(cfg)
    h = airg.setup(_sm(p), **prm)
    solve = airg.gmres_solve if cfg in (0, 4) else airg.richardson_solve
    res = solve(h, p.b, coarse_iterations=prm["coarse_iterations"])
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    A = sp.csr_matrix((p.vals, p.cols, p.row_offsets), shape=(p.n, p.n))
    rel = np.linalg.norm(p.b - A @ res.x) / np.linalg.norm(p.b)
    assert rel <= TOL_RES * 1.05
    assert h.n_levels >= 1


def test_edge_cases():
    a = airg.SparseMatrix.identity(10)
    h = airg.setup(a, coarse_size_target=100)
    res = airg.richardson_solve(h, np.zeros(10))
    assert res.stats.converged and res.stats.iterations == 0
    with pytest.raises(airg.InvalidArgument):
        airg.richardson_solve(h, np.zeros(9))
    with pytest.raises(airg.InvalidArgument):
        airg.DeviceCSR.upload(airg.SparseMatrix(1, 2, np.array([0, 2]), np.array([1, 0]), np.ones(2)))
    with pytest.raises(airg.InvalidArgument):
        airg.DeviceCSR.upload(airg.SparseMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([np.nan])))
    with pytest.raises(airg.InvalidArgument):
        airg.setup(a, cf=3)
    with pytest.raises(airg.AirgRuntimeError, match="stall"):  # test_air.cpp:280-291
        airg.setup(airg.SparseMatrix.identity(50), cf=1, ddc_enabled=0, coarse_size_target=5, poly_order=2)
    z = airg.SparseMatrix.from_triplets(3, 3, [(0, 0, 1.0), (0, 1, 2.0), (1, 0, 3.0), (2, 2, 1.0)])
    lab, _, _ = airg.cf_split(z, 0.5, 3, 0, ddc_enabled=True)
    assert set(np.unique(lab)) <= {0, 1}
    # batched split: empty batch, an empty matrix, and the same labels as one call
    assert airg.cf_split_batch_device([], [], ctx=h.ctx) == ([], [])
    e = airg.DeviceCSR.upload(airg.SparseMatrix(0, 0, np.array([0]), np.array([], np.int64), np.array([])))
    bl, br = airg.cf_split_batch_device([airg.DeviceCSR.upload(z), e], [0, 0])
    assert np.array_equal(bl[0].cpu().numpy()[:3], lab) and br[1].n_f == 0 and br[1].n_c == 0
    with pytest.raises(airg.InvalidArgument):
        airg.cf_split_batch_device([airg.DeviceCSR.upload(z)], [0], max_loops=0)


def test_solve_device_api_matches_host_api():
    import torch
    p = problems.make(0)
    prm = problems.setup_params(0)
    h = airg.setup(_sm(p), **prm)
    ctx = h.ctx
    tb = ctx.to_device(p.b)
    tx = ctx.empty(p.n, torch.float64)
    st, hist = h.solve_device(tb, tx, history_cap=64, coarse_iterations=3)
    res = airg.richardson_solve(h, p.b, coarse_iterations=3)
    assert same_bits(ctx.to_host(tx), res.x) and st.iterations == res.stats.iterations


def test_device_loop_history_realloc():
    """Two Richardson solves on one hierarchy with a growing max_iterations:
    the second reallocates the device history, which must rebuild the
    captured loop (the loop graph kept the freed buffer)."""
    p = problems.make(0)
    prm = problems.setup_params(0)
    h = airg.setup(_sm(p), **prm)
    r1 = airg.richardson_solve(h, p.b, coarse_iterations=3, max_iterations=3)
    assert not r1.stats.converged and r1.stats.iterations == 3 and len(r1.residual_history) == 4
    r2 = airg.richardson_solve(h, p.b, coarse_iterations=3, max_iterations=500)
    r3 = airg.richardson_solve(h, p.b, coarse_iterations=3)
    assert r2.stats.converged and r2.stats.iterations == r3.stats.iterations
    assert same_bits(r2.residual_history, r3.residual_history) and same_bits(r2.x, r3.x)
    np.testing.assert_allclose(r2.residual_history[:4], r1.residual_history, rtol=0, atol=0)
    assert r2.stats.final_relative_residual == r2.residual_history[-1] <= 1e-10
