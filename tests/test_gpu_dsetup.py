"""Owned-row distributed setup (airg_dist_setup_owned, SURVEY §8e "setup
collectives"): every rank builds and keeps only its rows of every level --
the CF split on the slabs, the A_ff halo rows gathered once for the
fixed-sparsity assembly, distance-2 halo rows of Aff^-1 and A P for Z and
R (A P), Gram matrix and growth norms reduced over the ranks, the coarse
rows moved to the next (halved) partition, the coarsest grid on rank 0.
Emulation mode (all P ranks in one process on one GPU, phase by phase).

Each row comes out of the single-GPU kernel on the same row in the same
entry order, so the hierarchy must equal the single-GPU setup's level for
level (labels, every block's size, coefficients, attempts) and the
distributed solve must reproduce the single-GPU solve."""
import glob
import os

import numpy as np
import pytest

from backends import same_bits
from paper_2408_08262_b200 import airg, problems

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
INT_FIELDS = ("n", "nnz", "n_f", "n_c", "n_f_pre", "ddc_converted", "nnz_ff", "nnz_fc", "nnz_cf",
              "nnz_ffinv", "nnz_r", "nnz_p", "poly_attempts", "effective_order")


def _params(g):
    return eval(str(g["params"][0]))


def _golden(path):
    g = np.load(path)
    n = len(g["rp"]) - 1
    return g, _params(g), airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])


def _compare_reports(h, d, exact_coeffs=True):
    assert d.n_levels == h.n_levels
    for l in range(h.n_levels):
        e, o = h.level(l), d.report(l)
        for f in INT_FIELDS:
            assert getattr(e, f) == getattr(o, f), (l, f, getattr(e, f), getattr(o, f))
        for f in ("alpha_diag", "max_theta_pre", "max_theta_post"):
            assert getattr(e, f) == getattr(o, f), (l, f)
        ce, co = np.array(e.coefficients), np.array(o.coefficients)
        if exact_coeffs:
            assert same_bits(ce, co), (l, ce, co)
        else:
            np.testing.assert_allclose(co, ce, rtol=1e-12, atol=0)
        assert abs(e.smoother_growth - o.smoother_growth) <= 1e-9 * abs(e.smoother_growth) + 1e-14, l
    hi, rc = h.info(), d.report(h.n_levels)
    assert (rc.n, rc.nnz, rc.nnz_ffinv) == (hi.coarse_n, hi.coarse_nnz, hi.coarse_inv_nnz)
    assert (rc.poly_attempts, rc.effective_order) == (hi.coarse_attempts, hi.coarse_effective_order)
    assert same_bits(np.array(rc.coefficients), np.array(hi.coarse_coefficients))


@pytest.mark.parametrize("path", GOLDEN[:4], ids=lambda p: os.path.basename(p)[:-4])
@pytest.mark.parametrize("P,threshold", [(1, 2.0), (2, 2.0), (3, 2.0), (4, 0.0), (8, 1e9)])
def test_owned_setup_matches_single_gpu(path, P, threshold):
    g, prm, a = _golden(path)
    h = airg.setup(a, **prm)
    d = airg.Dist.setup_owned(a, P, threshold=threshold, **prm)
    _compare_reports(h, d)
    # the same partitions and halving decisions as the distribution of the
    # global hierarchy (dist_create), from distributed locality counts
    dg = airg.Dist(h, P, threshold=threshold, starts=d._starts)
    for l in range(h.n_levels + 1):
        io, ig = d.level_info(l), dg.level_info(l)
        assert np.array_equal(io["starts"], ig["starts"]), l
        assert (io["active"], io["triggered"]) == (ig["active"], ig["triggered"]), l
        assert io["ratio_before"] == ig["ratio_before"] and io["ratio_after"] == ig["ratio_after"], l
        assert io["halo"] == ig["halo"], l
    ci = prm.get("coarse_iterations", 3)
    ref = airg.richardson_solve(h, g["b"], coarse_iterations=ci)
    res = d.solve(g["b"], coarse_iterations=ci)
    assert res.stats.converged and res.stats.iterations == ref.stats.iterations
    assert same_bits(res.x, ref.x), "owned-setup solve differs from the single-GPU solve"


@pytest.mark.parametrize("P", [2, 4])
def test_owned_setup_injected_bit_identical(P):
    """Coefficient injection: with the fit taken out, the
    owned hierarchy's operators are the single-GPU ones bit for bit, so the
    solve (Richardson and outer GMRES) is too."""
    g, prm, a = _golden(GOLDEN[1])
    h0 = airg.setup(a, **prm)
    inj = {"levels": [(list(h0.level(l).coefficients)[: prm.get("poly_order", 6) + 1],
                       h0.level(l).effective_order) for l in range(h0.n_levels)],
           "coarse": (list(h0.info().coarse_coefficients)[: prm.get("coarse_poly_order", 12) + 1],
                      h0.info().coarse_effective_order)}
    h = airg.setup(a, injection=inj, **prm)
    d = airg.Dist.setup_owned(a, P, injection=inj, **prm)
    assert d.n_levels == h.n_levels
    for l in range(h.n_levels):
        for f in INT_FIELDS:
            assert getattr(h.level(l), f) == getattr(d.report(l), f), (l, f)
    ci = prm.get("coarse_iterations", 3)
    for outer in (0, 1):
        ref = airg.richardson_solve(h, g["b"], coarse_iterations=ci, outer=outer)
        res = d.solve(g["b"], coarse_iterations=ci, outer=outer)
        assert res.stats.iterations == ref.stats.iterations, outer
        if outer == 0:
            assert same_bits(res.x, ref.x)
        else:  # dist GMRES sums its dots per rank, then over the ranks
            np.testing.assert_allclose(res.x, ref.x, rtol=1e-10, atol=1e-13)


def _c4(n_cells):
    p = problems.c4_tets_3d(n_cells, n_cells, n_cells)
    return p, airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)


@pytest.mark.parametrize("P", [2, 4])
def test_owned_setup_c4_zslabs(P):
    """C4 (the weak-scaling config) cut into z-slabs: the owned hierarchy
    equals the single-GPU one and the outer-GMRES solve converges to the
    same iterate."""
    p, a = _c4(12)
    prm = dict(problems.setup_params(4), coarse_size_target=400)
    h = airg.setup(a, **prm)
    starts = np.linspace(0, p.n, P + 1).astype(np.int64)
    d = airg.Dist.setup_owned(a, P, starts=starts, **prm)
    _compare_reports(h, d)
    ref = airg.richardson_solve(h, p.b, coarse_iterations=3, outer=1, max_iterations=200)
    res = d.solve(p.b, coarse_iterations=3, outer=1, max_iterations=200)
    assert res.stats.converged and abs(res.stats.iterations - ref.stats.iterations) <= 1
    np.testing.assert_allclose(res.x, ref.x, rtol=1e-8 * np.abs(ref.x).max(), atol=1e-12)


@pytest.mark.parametrize("P,threshold", [(2, 2.0), (3, 1e9), (4, 2.0)])
def test_owned_setup_fast_mode(P, threshold):
    """The owned setup builds the fast V-cycle's A_F P and W_2 slabs from halo
    rows (dsetup.cu): the same products in the same order as one GPU, so the
    distributed fast solve equals the fast solve of the distributed global
    hierarchy (dist_create slicing the one-GPU operators) bit for bit, and
    the one-GPU fast solve to the parity tolerance."""
    p, a = _c4(12)
    prm = dict(problems.setup_params(4), coarse_size_target=400, fused_smooths=2)
    h = airg.setup(a, **prm)
    starts = np.linspace(0, p.n, P + 1).astype(np.int64)
    d = airg.Dist.setup_owned(a, P, starts=starts, threshold=threshold, **prm)
    dg = airg.Dist(h, P, threshold=threshold, starts=d._starts)
    for outer in (0, 1):
        kw = dict(coarse_iterations=3, outer=outer, max_iterations=300, fast=1)
        res = d.solve(p.b, **kw)
        rg = dg.solve(p.b, **kw)
        ref = airg.richardson_solve(h, p.b, **kw)
        assert res.stats.converged and res.stats.final_relative_residual <= 1e-10
        assert same_bits(res.x, rg.x) and res.stats.iterations == rg.stats.iterations
        assert abs(res.stats.iterations - ref.stats.iterations) <= 1
        assert np.linalg.norm(res.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


@pytest.mark.parametrize("smooths", [0, 1])
def test_owned_setup_fast_mode_other_smooth_counts(smooths):
    """W_0 (empty: x = P e_c) and W_1 = Q on the slabs: the distributed fast
    V-cycle with up_f_smooths 0 / 1 matches the one-GPU fast solve."""
    p, a = _c4(10)
    prm = dict(problems.setup_params(4), coarse_size_target=400, fused_smooths=smooths)
    h = airg.setup(a, **prm)
    starts = np.linspace(0, p.n, 4).astype(np.int64)
    d = airg.Dist.setup_owned(a, 3, starts=starts, **prm)
    dg = airg.Dist(h, 3, starts=d._starts)
    kw = dict(coarse_iterations=3, outer=1, max_iterations=400, fast=1, up_f_smooths=smooths)
    res = d.solve(p.b, **kw)
    rg = dg.solve(p.b, **kw)
    ref = airg.richardson_solve(h, p.b, **kw)
    assert same_bits(res.x, rg.x) and res.stats.iterations == rg.stats.iterations
    if smooths == 0:  # V(0,0) (no F-smoothing) does not converge here -- on one GPU either
        assert not res.stats.converged and not ref.stats.converged
        return
    assert res.stats.converged
    assert abs(res.stats.iterations - ref.stats.iterations) <= 1
    assert np.linalg.norm(res.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


def test_owned_setup_memory_partitioned():
    """No rank holds a level operator: at P = 4 each rank's resident bytes
    are about a quarter of one rank's at P = 1 (plus halos and the gathered
    coarsest grid on rank 0)."""
    p = problems.c2_structured_3d(32)
    prm = dict(problems.setup_params(2), coarse_size_target=500)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    one = airg.Dist.setup_owned(a, 1, **prm).rank_bytes(0)
    d = airg.Dist.setup_owned(a, 4, threshold=0.0, **prm)
    per = [d.rank_bytes(r) for r in range(4)]
    assert max(per) < 0.4 * one, (per, one)
    assert sum(per) < 1.25 * one, (per, one)


def test_owned_setup_nccl_single_rank():
    """The NCCL code path of the owned setup (rank >= 0, a communicator,
    all-gathered counts, the request/response row gathers) on a 1-rank
    communicator."""
    g, prm, a = _golden(GOLDEN[0])
    h = airg.setup(a, **prm)
    comm = airg.NcclComm(1, 0, airg.nccl_unique_id())
    d = airg.Dist.setup_owned(a, 1, rank=0, comm=comm, **prm)
    _compare_reports(h, d)
    ref = airg.richardson_solve(h, g["b"], coarse_iterations=3)
    tb = h.ctx.to_device(g["b"])
    tx = h.ctx.empty(len(g["b"]), h.ctx.torch.float64)
    st, _ = d.solve_device(tb, tx, coarse_iterations=3)
    assert st.iterations == ref.stats.iterations and same_bits(h.ctx.to_host(tx), ref.x)


def test_owned_setup_rejects_unsupported():
    g, prm, a = _golden(GOLDEN[0])
    with pytest.raises(airg.InvalidArgument):
        airg.Dist.setup_owned(a, 2, **dict(prm, sparsity_order=2))
    with pytest.raises(airg.InvalidArgument):
        airg.Dist.setup_owned(a, 2, **dict(prm, cf=1))
    with pytest.raises(airg.InvalidArgument):
        airg.Dist.setup_owned(a, 2, starts=np.array([0, 5, 3]), **prm)
