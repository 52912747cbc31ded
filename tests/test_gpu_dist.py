"""Multi-GPU path on one GPU: the row-slab distributed solve in
emulation mode (all P ranks in one process, run phase by phase; halos moved
by a gather kernel). Because only column indices are remapped and every row
keeps its entry order, the distributed V-cycle reproduces the single-GPU
solution bit for bit, for any P and any halving schedule."""
import glob
import os

import numpy as np
import pytest

from backends import same_bits
from paper_2408_08262_b200 import airg, problems

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _params(g):
    return eval(str(g["params"][0]))


@pytest.mark.parametrize("path", GOLDEN[:4], ids=lambda p: os.path.basename(p)[:-4])
@pytest.mark.parametrize("P,threshold", [(2, 2.0), (3, 2.0), (4, 0.0), (8, 1e9)])
def test_dist_emulated_bit_identical(path, P, threshold):
    g = np.load(path)
    prm = _params(g)
    n = len(g["rp"]) - 1
    h = airg.setup(airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]), **prm)
    ci = prm.get("coarse_iterations", 3)
    ref = airg.richardson_solve(h, g["b"], coarse_iterations=ci)
    d = airg.Dist(h, P, threshold=threshold)
    res = d.solve(g["b"], coarse_iterations=ci)
    assert res.stats.converged and res.stats.iterations == ref.stats.iterations
    assert same_bits(res.x, ref.x), "distributed solve differs from the single-GPU solve"
    np.testing.assert_allclose(res.residual_history, ref.residual_history, rtol=1e-9, atol=1e-15)
    # partitions: contiguous, monotone, cover the level; halving follows the rule
    active = P
    for l in range(h.n_levels):
        info = d.level_info(l)
        s = info["starts"]
        assert s[0] == 0 and s[-1] == h.level(l).n and (np.diff(s) >= 0).all()
        if info["triggered"]:
            assert info["ratio_before"] < threshold and info["active"] == (active + 1) // 2
        active = info["active"]
        assert (np.diff(s) > 0).sum() <= active
    top = d.level_info(h.n_levels)
    assert top["active"] == 1 and top["starts"][1] == h.info().coarse_n  # gathered on rank 0


def test_dist_nccl_single_rank_path():
    """The NCCL transport code path (rank >= 0, communicator, allreduced
    norms) on a 1-rank communicator: only one GPU is available to the run,
    and ranks that wait on each other must not share a GPU."""
    g = np.load(GOLDEN[0])
    prm = _params(g)
    n = len(g["rp"]) - 1
    h = airg.setup(airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]), **prm)
    ref = airg.richardson_solve(h, g["b"], coarse_iterations=3)
    comm = airg.NcclComm(1, 0, airg.nccl_unique_id())
    d = airg.Dist(h, 1, rank=0, comm=comm)
    tb = h.ctx.to_device(g["b"])
    tx = h.ctx.empty(n, h.ctx.torch.float64)
    st, _ = d.solve_device(tb, tx, coarse_iterations=3)
    assert st.iterations == ref.stats.iterations and same_bits(h.ctx.to_host(tx), ref.x)


def test_c2_stacked_family_matches_c2():
    a = problems.c2_structured_3d(16)
    b = problems._c2_stacked(16, 0, 1)
    assert np.array_equal(a.cols, b.cols) and same_bits(a.vals, b.vals)


def test_dist_c2_reduced_with_zslabs():
    p = problems.c2_structured_3d(32)
    prm = dict(problems.setup_params(2), coarse_size_target=500)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ref = airg.richardson_solve(h, p.b, coarse_iterations=3)
    starts = np.linspace(0, p.n, 5).astype(np.int64)  # z-slabs of 8 planes
    d = airg.Dist(h, 4, threshold=2.0, starts=starts)
    assert d.transport == ("p2p" if os.environ.get("AIRG_TRANSPORT") == "p2p" else "gather")
    res = d.solve(p.b, coarse_iterations=3)
    assert same_bits(res.x, ref.x)
    assert d.level_info(0)["halo"] > 0


@pytest.mark.parametrize("min_rows", [1000, 6000])
def test_dist_min_rows_rule_bit_identical(min_rows, monkeypatch):
    """AIRG_DIST_MIN_ROWS (the latency rule for NVLink, dist.cu) halves the
    active ranks on the small levels; the solve keeps the one-GPU bits."""
    monkeypatch.setenv("AIRG_DIST_MIN_ROWS", str(min_rows))
    p = problems.c2_structured_3d(32)
    prm = dict(problems.setup_params(2), coarse_size_target=500)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ref = airg.richardson_solve(h, p.b, coarse_iterations=3)
    d = airg.Dist(h, 8, threshold=2.0, starts=np.linspace(0, p.n, 9).astype(np.int64))
    act = [d.level_info(l)["active"] for l in range(h.n_levels)]
    assert act == sorted(act, reverse=True) and act[-1] < 8
    # level 0 keeps the caller's slabs (its b / x buffers); the rule applies below
    assert act[0] == 8
    for l in range(1, h.n_levels):
        assert h.level(l).n >= min_rows * d.level_info(l)["active"] or d.level_info(l)["active"] == 1
    res = d.solve(p.b, coarse_iterations=3)
    assert same_bits(res.x, ref.x)


def _split_cases():
    out = []
    for path in GOLDEN[:4]:
        g = np.load(path)
        prm = _params(g)
        n = len(g["rp"]) - 1
        out.append((os.path.basename(path)[:-4], airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]),
                    prm.get("strength_alpha", 0.5)))
    p = problems.c2_structured_3d(32)
    out.append(("c2_32", airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), 0.5))
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("ddc", [True, False])
def test_dist_cf_split_matches_single_gpu(P, ddc):
    """Row-slab PMISR-DDC (halo weights, reverse-summed |S^T| and 'not
    minimal' marks, allreduced DDC histogram) == the one-GPU split, bitwise."""
    rng = np.random.default_rng(P)
    for name, a, alpha in _split_cases():
        n = a.nrows
        for seed in (0, 7):
            lab, _, rep = airg.cf_split(a, alpha, 3, seed, ddc_enabled=ddc)
            if P > 1 and seed == 7:  # ragged slabs, some empty
                cuts = np.sort(rng.integers(0, n + 1, P - 1))
                starts = np.concatenate([[0], cuts, [n]])
            else:
                starts = None
            dl, drep = airg.dist_cf_split(a, P, starts=starts, alpha=alpha, seed=seed, ddc_enabled=ddc)
            assert np.array_equal(dl, lab), f"{name} P={P} seed={seed}: labels differ"
            assert (drep.n_f_pre, drep.n_f, drep.n_converted, drep.s_nnz) == \
                (rep.n_f_pre, rep.n_f, rep.n_converted, rep.s_nnz), name
            assert same_bits(np.float64([drep.max_theta, drep.alpha_diag]),
                             np.float64([rep.max_theta, rep.alpha_diag])), name


def test_dist_cf_split_nccl_single_rank():
    p = problems.c2_structured_3d(24)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    lab, _, _ = airg.cf_split(a, 0.5, 3, 3)
    ctx = airg.default_context()
    d = airg.DeviceCSR.upload(a, ctx)
    comm = airg.NcclComm(1, 0, airg.nccl_unique_id())
    tl, _ = airg.dist_cf_split_device(d, [0, p.n], rank=0, comm=comm, seed=3)
    assert np.array_equal(ctx.to_host(tl)[: p.n], lab)


def _hier_digest(h):
    """Every level matrix, label vector and coefficient set of a hierarchy."""
    import hashlib
    d = hashlib.sha256()
    info = h.info()
    for l in range(h.n_levels):
        lv = h.level(l)
        d.update(np.asarray(lv.coefficients[:8]).tobytes())
        d.update(h.labels(l).tobytes())
        for w in ("a", "a_ff", "a_fc", "a_cf", "ff_inv", "r", "p"):
            m = h.matrix(l, w)
            d.update(m.row_offsets.tobytes())
            d.update(m.col_indices.tobytes())
            d.update(m.values.tobytes())
    d.update(np.asarray(info.coarse_coefficients[:16]).tobytes())
    return d.hexdigest()


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_dist_setup_bit_identical(P):
    """Row work of the setup split over P emulated ranks (CF split on row
    slabs, gathered SpGEMM / assembly / SpMV slabs): the same hierarchy bit for
    bit as the one-GPU setup, native coefficients included."""
    for path in GOLDEN[:4]:
        g = np.load(path)
        prm = _params(g)
        n = len(g["rp"]) - 1
        a = airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"])
        ref = airg.setup(a, **prm)
        h = airg.setup(a, nranks=P, **prm)
        assert _hier_digest(h) == _hier_digest(ref), f"{os.path.basename(path)} P={P}"
    p = problems.c2_structured_3d(24)
    prm = dict(problems.setup_params(2), coarse_size_target=300)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    assert _hier_digest(airg.setup(a, nranks=P, **prm)) == _hier_digest(airg.setup(a, **prm))


def test_dist_setup_nccl_single_rank_then_solve():
    p = problems.c2_structured_3d(24)
    prm = dict(problems.setup_params(2), coarse_size_target=300)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    ref = airg.setup(a, **prm)
    comm = airg.NcclComm(1, 0, airg.nccl_unique_id())
    h = airg.setup(a, nranks=1, rank=0, comm=comm, **prm)
    assert _hier_digest(h) == _hier_digest(ref)
    d = airg.Dist(h, 1, rank=0, comm=comm)
    tb = h.ctx.to_device(p.b)
    tx = h.ctx.empty(p.n, h.ctx.torch.float64)
    st, _ = d.solve_device(tb, tx, coarse_iterations=3)
    r0 = airg.richardson_solve(ref, p.b, coarse_iterations=3)
    assert st.iterations == r0.stats.iterations and same_bits(h.ctx.to_host(tx), r0.x)


P2P_SCRIPT = r"""
import glob, os, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
gold = sorted(glob.glob(os.path.join(%r, "golden", "*.npz")))[:4]
cases = []
for path in gold:
    g = np.load(path)
    prm = eval(str(g["params"][0]))
    n = len(g["rp"]) - 1
    cases.append((airg.SparseMatrix.from_arrays(n, n, g["rp"], g["ci"], g["v"]), prm, g["b"], None))
p = problems.c2_structured_3d(32)
cases.append((airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals),
              dict(problems.setup_params(2), coarse_size_target=500), p.b, np.linspace(0, p.n, 5).astype(np.int64)))
for a, prm, b, starts in cases:
    h = airg.setup(a, **prm)
    ci = prm.get("coarse_iterations", 3)
    ref = airg.richardson_solve(h, b, coarse_iterations=ci)
    for P, thr in ((2, 2.0), (3, 2.0), (4, 0.0), (8, 1e9)):
        if starts is not None and P != 4:
            continue
        d = airg.Dist(h, P, threshold=thr, starts=starts)
        assert d.transport == "p2p"
        for rep in range(2):  # the slot counters carry over between solves
            res = d.solve(b, coarse_iterations=ci)
            assert res.stats.iterations == ref.stats.iterations, (P, rep)
            assert res.x.tobytes() == ref.x.tobytes(), (P, rep)
print("p2p ok")
""" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))


def test_dist_p2p_transport_emulated_bit_identical():
    """AIRG_TRANSPORT=p2p: halo entries pushed into the consumers' halo slots
    of the per-rank arenas with delivery / consumption counters (the NVLink
    peer-store protocol, halo_p2p.cu), all ranks emulated on one GPU: same
    bits as one GPU, twice in a row on the same distribution."""
    import subprocess
    import sys
    for extra in ({}, {"AIRG_DIST_MIN_ROWS": "3000"}):  # slabs as given / merged on the small levels
        env = dict(os.environ, AIRG_TRANSPORT="p2p", **extra)
        out = subprocess.run([sys.executable, "-c", P2P_SCRIPT], env=env, capture_output=True, text=True,
                             timeout=900)
        assert out.returncode == 0, out.stderr[-3000:]
        assert "p2p ok" in out.stdout


@pytest.mark.parametrize("P,threshold", [(2, 2.0), (3, 2.0), (4, 1e9)])
def test_dist_gmres_emulated_matches_one_gpu(P, threshold):
    """The outer GMRES(30) over the row slabs (dist.cu dist_gmres; the C4
    solver of the weak-scaling bench): the V-cycle is bit-identical to one
    GPU's, the inner products are slab partials + one allreduce, so the solve
    agrees with the one-GPU GMRES to the parity tolerance."""
    import scipy.sparse as sp
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=500)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ref = airg.gmres_solve(h, p.b, coarse_iterations=3)
    d = airg.Dist(h, P, threshold=threshold)
    res = d.solve(p.b, coarse_iterations=3, outer=1, gmres_restart=30)
    assert res.stats.converged and res.stats.final_relative_residual <= 1e-10
    assert abs(res.stats.iterations - ref.stats.iterations) <= 1
    assert np.linalg.norm(res.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    A = sp.csr_matrix((p.vals, p.cols, p.row_offsets), shape=(p.n, p.n))
    assert np.linalg.norm(p.b - A @ res.x) <= 1.05e-10 * np.linalg.norm(p.b)


@pytest.mark.parametrize("P,threshold", [(2, 2.0), (3, 1e9), (4, 2.0)])
def test_dist_fast_mode_emulated_matches_one_gpu(P, threshold):
    """The fast V-cycle on the row slabs (dist.cu: lane-group rows and the
    fused A_F P / W_k operators sliced by F rows, their halos planned with the
    other operators'): Richardson and GMRES(30) agree with the one-GPU fast
    solves to the parity tolerance, and differ from the exact distributed
    solve (which is the one-GPU exact solve bit for bit)."""
    import scipy.sparse as sp
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=500, fused_smooths=2)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    A = sp.csr_matrix((p.vals, p.cols, p.row_offsets), shape=(p.n, p.n))
    d = airg.Dist(h, P, threshold=threshold)
    for outer in (0, 1):
        kw = dict(coarse_iterations=3, outer=outer, gmres_restart=30, max_iterations=300)
        ref = airg.richardson_solve(h, p.b, fast=1, **kw)
        res = d.solve(p.b, fast=1, **kw)
        ex = d.solve(p.b, **kw)
        assert res.stats.converged and res.stats.final_relative_residual <= 1e-10
        assert abs(res.stats.iterations - ref.stats.iterations) <= 1
        assert np.linalg.norm(res.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
        assert np.linalg.norm(p.b - A @ res.x) <= 1.05e-10 * np.linalg.norm(p.b)
        assert not np.array_equal(res.x.view(np.uint64), ex.x.view(np.uint64))


def test_dist_gmres_nccl_single_rank_path():
    """The NCCL code path of the distributed GMRES (allreduced dots) on a
    1-rank communicator (one GPU in this run)."""
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=500)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ref = airg.gmres_solve(h, p.b, coarse_iterations=3)
    comm = airg.NcclComm(1, 0, airg.nccl_unique_id())
    d = airg.Dist(h, 1, rank=0, comm=comm)
    tb = h.ctx.to_device(p.b)
    tx = h.ctx.empty(p.n, h.ctx.torch.float64)
    st, _ = d.solve_device(tb, tx, coarse_iterations=3, outer=1)
    x = h.ctx.to_host(tx)
    assert st.converged and abs(st.iterations - ref.stats.iterations) <= 1
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


def test_dist_halo_bytes_accounting():
    """The NVLink bytes the N > 1 bench reports: per V-cycle, every exchange
    of enqueue_vcycle counted from the halo plans (8 B per halo entry)."""
    p = problems.c2_structured_3d(24)
    prm = dict(problems.setup_params(2), coarse_size_target=300)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    one = airg.Dist(h, 1)
    assert one.halo_bytes(coarse_iterations=3) == (0, 0)
    d = airg.Dist(h, 4, threshold=0.0, starts=np.linspace(0, p.n, 5).astype(np.int64))
    v, s = d.halo_bytes(coarse_iterations=3)
    # the level-0 SpMV reads one upwind plane of 24 x 24 cells across each of
    # the three slab boundaries (one-sided halo)
    assert s == 8 * 3 * 24 * 24
    assert v > s and v % 8 == 0 and v >= 8 * d.level_info(0)["halo"]


def test_dist_owns_its_slabs_and_memory_scales():
    """Each rank of a distribution holds only its slabs (operators, maps,
    vectors; the coarsest grid on rank 0): with 4 ranks the largest share is
    well under half of the one-rank total, and the global hierarchy can be
    freed -- the solve still gives the one-GPU bits."""
    p = problems.c2_structured_3d(24)
    prm = dict(problems.setup_params(2), coarse_size_target=300)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ref = airg.richardson_solve(h, p.b, coarse_iterations=3)
    one = airg.Dist(h, 1).rank_bytes(0)
    d = airg.Dist(h, 4, threshold=0.0, starts=np.linspace(0, p.n, 5).astype(np.int64))
    shares = [d.rank_bytes(r) for r in range(4)]
    assert max(shares) < 0.4 * one and sum(shares) < 1.3 * one, (shares, one)
    d.release_hierarchy()
    h.close()
    del h
    res = d.solve(p.b, coarse_iterations=3)
    assert res.stats.iterations == ref.stats.iterations and same_bits(res.x, ref.x)


@pytest.mark.skipif(__import__("torch").cuda.device_count() < 2, reason="needs two GPUs (one process per GPU)")
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_two_process_nccl_and_p2p_match_one_gpu(transport):
    """One process per GPU over a real communicator: the NCCL and the NVLink
    peer-store (p2p) transports, two consecutive Richardson solves bit-identical
    to one GPU, and the distributed GMRES within the parity tolerance
    (the p2p path had only run in emulation)."""
    import subprocess
    import sys
    env = dict(os.environ)
    if transport == "p2p":
        env["AIRG_TRANSPORT"] = "p2p"
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpu2_dist_worker.py")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", "29571", worker],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "RESULT 1" in out.stdout, out.stdout[-2000:]
