"""Full-size parity against the REFERENCE (SURVEY §8c P1/P2/P4/P5 at the
BASELINE.json sizes of C1-C4), through the C-ABI.

The fixtures tests/golden/full/c{1,2,3,4}.npz come from the compiled
reference (oracle/_ref) run at full size by tests/golden/make_full.py (the
GPU box has no /root/reference, and the serial setup of C3 alone takes
minutes). Per config:

* the generator reproduces the reference's input bit for bit (digest);
* NATIVE setup (GPU double-double coefficient fit): the same level count,
  per-level sizes, DDC conversions, effective orders and attempt counts as
  the reference, every level's labels bit-identical (sha256), growth factors
  on the same side of the 0.5 acceptance bound and within 1e-6 relative,
  coefficients within 1e-7 relative;
* INJECTION setup (the reference's coefficients): every matrix of every
  level bit-identical (sha256 of the seven level matrices), and for the
  Richardson configs the solve bit-identical (sha256 of x, iteration count);
* NATIVE solve: converged to rtol 1e-10 by a fresh host matvec,
  iterations within +-1 of the reference, solution within 1e-8 relative L2
  of the reference's -- over the full vector against the injection-mode
  solution (bit-identical to the reference's x, checked by digest, for
  Richardson) and on 65,536 seeded indices against the reference's own x.
C4 runs the outer GMRES(30) in both: the reference's Richardson diverges
there (fixture `c4_richardson_history`), as the GPU's does.
"""
import glob
import hashlib
import os

import numpy as np
import pytest

from paper_2408_08262_b200 import airg, problems

pytestmark = pytest.mark.gpu
FULL = os.path.join(os.path.dirname(__file__), "golden", "full")
TOL_X = 1e-8
TOL_RES = 1e-10
CONFIGS = [1, 2, 3, 4]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _problem_digest(p):
    h = hashlib.sha256()
    for a in (np.asarray(p.row_offsets, np.int64), np.asarray(p.cols, np.int64),
              np.asarray(p.vals, np.float64), np.asarray(p.b, np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _mat_digest(m):
    return _digest(np.concatenate([np.asarray(m.row_offsets, np.int64).view(np.uint8),
                                   np.asarray(m.col_indices, np.int64).view(np.uint8),
                                   np.asarray(m.values, np.float64).view(np.uint8)]))


_xinj = {}  # injection-mode solutions, by config


@pytest.fixture(scope="module", params=CONFIGS, ids=lambda c: f"C{c}")
def case(request):
    """(fixture, problem) of one config; module scope groups the tests by
    config, so each full-size system is generated once."""
    cfg = request.param
    g = dict(np.load(os.path.join(FULL, f"c{cfg}.npz")))
    return cfg, g, problems.make(cfg)


def _injection(g, prm):
    nl = int(g["n_levels"])
    return {"levels": [(list(g["level_coeffs"][l]), int(g["level_eff"][l])) for l in range(nl)],
            "coarse": (list(g["coarse_coeffs"]), int(g["coarse_eff"]))}


def _host_rel(p, x):
    import scipy.sparse as sp
    A = sp.csr_matrix((p.vals, p.cols, p.row_offsets), shape=(p.n, p.n))
    return np.linalg.norm(p.b - A @ x) / np.linalg.norm(p.b)


def test_full_native_setup_matches_reference(case):
    cfg, g, p = case
    assert _problem_digest(p) == str(g["problem_digest"]), "generator drifted from the fixture's input"
    prm = eval(str(g["params"][0]))
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    nl = int(g["n_levels"])
    assert h.n_levels == nl
    info = h.info()
    assert info.coarse_n == int(g["coarse_n"]) and info.coarse_nnz == int(g["coarse_nnz"])
    assert info.coarse_effective_order == int(g["coarse_eff"])
    for l in range(nl):
        L = h.level(l)
        assert (L.n, L.nnz, L.n_f, L.n_c, L.ddc_converted) == (
            g["level_n"][l], g["level_nnz"][l], g["level_nf"][l], g["level_nc"][l], g["level_conv"][l]), l
        assert L.effective_order == g["level_eff"][l], l
        assert L.poly_attempts == g["level_attempts"][l], l
        gr, go = L.smoother_growth, float(g["level_growth"][l])
        assert (gr <= 0.5) == (go <= 0.5), (l, gr, go)
        assert abs(gr - go) <= 1e-6 * abs(go) + 1e-12, (l, gr, go)
        c1 = np.array(L.coefficients[: prm["poly_order"] + 1])
        c2 = g["level_coeffs"][l]
        assert np.abs(c1 - c2).max() <= 1e-7 * max(1.0, np.abs(c2).max()), l
        assert _digest(h.labels(l)) == str(g["level_labels_digest"][l]), f"labels of level {l}"


def test_full_injected_hierarchy_and_solve_bit_identical(case):
    cfg, g, p = case
    prm = eval(str(g["params"][0]))
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals),
                   injection=_injection(g, prm), **prm)
    nl = int(g["n_levels"])
    assert h.n_levels == nl
    for l in range(nl):
        assert _digest(h.labels(l)) == str(g["level_labels_digest"][l]), l
        got = "|".join(_mat_digest(h.matrix(l, w)) for w in range(7))
        assert got == str(g["level_matrix_digest"][l]), f"level {l} matrices differ"
    ci = prm["coarse_iterations"]
    if int(g["outer"]):
        res = airg.gmres_solve(h, p.b, coarse_iterations=ci, max_iterations=400)
        assert abs(res.stats.iterations - int(g["solve"][0])) <= 1
        idx = g["x_index"]
        assert np.linalg.norm(res.x[idx] - g["x_sample"]) <= TOL_X * np.linalg.norm(g["x_sample"])
    else:
        res = airg.richardson_solve(h, p.b, coarse_iterations=ci, max_iterations=400)
        assert res.stats.iterations == int(g["solve"][0])
        assert _digest(res.x) == str(g["x_digest"]), "Richardson solution not bit-identical to the reference"
    assert res.stats.converged and _host_rel(p, res.x) <= TOL_RES * 1.05
    _xinj[cfg] = res.x


def test_full_native_solve_within_tolerance(case):
    cfg, g, p = case
    prm = eval(str(g["params"][0]))
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ci = prm["coarse_iterations"]
    fn = airg.gmres_solve if int(g["outer"]) else airg.richardson_solve
    res = fn(h, p.b, coarse_iterations=ci, max_iterations=400)
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    assert _host_rel(p, res.x) <= TOL_RES * 1.05
    assert abs(res.stats.iterations - int(g["solve"][0])) <= 1
    idx = g["x_index"]
    assert np.linalg.norm(res.x[idx] - g["x_sample"]) <= TOL_X * np.linalg.norm(g["x_sample"])
    xr = _xinj.get(cfg)
    if xr is None:  # the injection-mode solution (bit-identical to the reference's for Richardson)
        hi = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals),
                        injection=_injection(g, prm), **prm)
        xr = fn(hi, p.b, coarse_iterations=ci, max_iterations=400).x
    assert np.linalg.norm(res.x - xr) <= TOL_X * np.linalg.norm(xr)
    assert abs(np.linalg.norm(xr) - float(g["x_norm"])) <= 1e-8 * float(g["x_norm"])


def test_c4_reference_richardson_diverges(case):
    """The reason C4 runs the outer GMRES: the reference's own Richardson on
    the full-size C4 hierarchy grows the residual (level-0 smoother growth
    2.33 on the best of six attempts), and so does the GPU's."""
    cfg, g, p = case
    if cfg != 4:
        pytest.skip("C4 only")
    rh = g["c4_richardson_history"]
    assert rh[-1] > 1e3 and float(g["level_growth"][0]) > 0.5
    prm = eval(str(g["params"][0]))
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals),
                   injection=_injection(g, prm), **prm)
    res = airg.richardson_solve(h, p.b, coarse_iterations=prm["coarse_iterations"], max_iterations=len(rh) - 1)
    assert not res.stats.converged
    np.testing.assert_allclose(res.residual_history, rh, rtol=1e-6)


def test_full_fast_mode_solve_within_tolerance(case):
    """The bench's configuration (fast mode: lane-group rows with FMA, the
    fused level operators built at setup, Gram-corrected CGS2 in the device
    GMRES) against the REFERENCE's full-size solve: converged to 1e-10 by a
    fresh host matvec, iterations within +-1, x within 1e-8 (sampled entries
    against the reference's own x, full vector against the injection-mode x)."""
    cfg, g, p = case
    prm = dict(eval(str(g["params"][0])), fused_smooths=2)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    fn = airg.gmres_solve if int(g["outer"]) else airg.richardson_solve
    res = fn(h, p.b, coarse_iterations=prm["coarse_iterations"], max_iterations=400, fast=1)
    assert res.stats.converged and res.stats.final_relative_residual <= TOL_RES
    assert _host_rel(p, res.x) <= TOL_RES * 1.05
    assert abs(res.stats.iterations - int(g["solve"][0])) <= 1, (res.stats.iterations, int(g["solve"][0]))
    idx = g["x_index"]
    assert np.linalg.norm(res.x[idx] - g["x_sample"]) <= TOL_X * np.linalg.norm(g["x_sample"])
    xr = _xinj.get(cfg)
    if xr is not None:
        assert np.linalg.norm(res.x - xr) <= TOL_X * np.linalg.norm(xr)
