"""Launch-mode and arithmetic-mode invariants of the solve (tiled.cuh).

* EXACT mode gives the same bits with and without programmatic dependent
  launch and with the host-driven instead of the graph-resident loop
  (environment switches read once per process, hence one subprocess each).
* FAST mode (lane groups, FMA, tree reductions) solves within the parity
  tolerance of the exact mode (rtol 1e-10, +-1 iteration, 1e-8 in x) and is
  deterministic run to run.
* The fused CF split's row-load variants give the step-by-step split's
  labels and DDC reports on every level.
"""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2408_08262_b200 import airg, problems

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
p = problems.c2_structured_3d(24)
prm = dict(problems.setup_params(2), coarse_size_target=300)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(a, **prm)
r = airg.richardson_solve(h, p.b, coarse_iterations=3)
y = airg.spmv(h.matrix(1, 0), np.random.default_rng(0).random(h.level(1).n))
print(r.stats.iterations, hashlib.sha256(r.x.tobytes()).hexdigest(), hashlib.sha256(y.tobytes()).hexdigest())
""" % REPO

MODES = {"default": {}, "nopdl": {"AIRG_PDL": "0"}, "host_loop": {"AIRG_DEVLOOP": "0"}}


def _run(script, env_extra, keys):
    env = dict(os.environ)
    for k in keys:
        env.pop(k, None)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.strip().split("\n")[-1]


def test_exact_launch_modes_bit_identical():
    keys = ("AIRG_PDL", "AIRG_DEVLOOP")
    base = _run(SCRIPT, MODES["default"], keys)
    for name, env in MODES.items():
        assert _run(SCRIPT, env, keys) == base, f"launch mode {name} changes the bits"


@pytest.mark.parametrize("cfg,scale,outer", [(1, 0.25, 0), (2, 0.25, 0), (3, 0.125, 0), (4, 0.5, 1), (0, 1.0, 1)])
def test_fast_mode_within_tolerance(cfg, scale, outer):
    p = problems.make(cfg, scale)
    prm = problems.setup_params(cfg)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    kw = dict(coarse_iterations=prm["coarse_iterations"], outer=outer, max_iterations=400)
    ex = airg.richardson_solve(h, p.b, **kw)
    fa = airg.richardson_solve(h, p.b, fast=1, **kw)
    fb = airg.richardson_solve(h, p.b, fast=1, **kw)
    assert ex.stats.converged and fa.stats.converged
    assert fa.stats.final_relative_residual <= 1e-10
    assert abs(fa.stats.iterations - ex.stats.iterations) <= 1
    assert np.linalg.norm(fa.x - ex.x) <= 1e-8 * np.linalg.norm(ex.x)
    assert hashlib.sha256(fa.x.tobytes()).digest() == hashlib.sha256(fb.x.tobytes()).digest(), \
        "fast mode is not deterministic"
    import scipy.sparse as sp
    A = sp.csr_matrix((p.vals, p.cols, p.row_offsets), shape=(p.n, p.n))
    assert np.linalg.norm(p.b - A @ fa.x) <= 1.05e-10 * np.linalg.norm(p.b)


def test_fast_vcycle_close_to_exact():
    """One fast V-cycle against the exact (reference-bit) V-cycle: the same
    operator up to rounding."""
    p = problems.make(4, 0.5)
    prm = problems.setup_params(4)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ve = h.vcycle(p.b, coarse_iterations=3)
    vf = h.vcycle(p.b, coarse_iterations=3, fast=1)
    assert np.linalg.norm(vf - ve) <= 1e-12 * np.linalg.norm(ve)


CF_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
out = []
for cfg, scale in ((2, 0.1875), (3, 0.125), (4, 0.25)):
    p = problems.make(cfg, scale)
    prm = dict(problems.setup_params(cfg), coarse_size_target=300)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    lab = np.concatenate([h.labels(l) for l in range(h.n_levels)])
    reps = [(h.level(l).max_theta_pre, h.level(l).alpha_diag, h.level(l).ddc_converted) for l in range(h.n_levels)]
    out.append(hashlib.sha256(lab.tobytes() + repr(reps).encode()).hexdigest()[:16])
print(" ".join(out))
""" % REPO

CF_VARIANTS = {
    "legacy": {"AIRG_CF": "legacy"},
    "fused_scalar": {"AIRG_CF_VEC": "100000"},
    "fused_vec": {"AIRG_CF_VEC": "1"},
    "fused_default": {},
}


def test_cf_split_variants_bit_identical():
    """The fused split (scalar or 16-byte row loads) and the step-by-step
    split give the same hierarchy labels and DDC reports on every level
    (C2/C3/C4, reduced)."""
    keys = ("AIRG_CF", "AIRG_CF_VEC")
    base = _run(CF_SCRIPT, CF_VARIANTS["legacy"], keys)
    for name, env in CF_VARIANTS.items():
        if name != "legacy":
            assert _run(CF_SCRIPT, env, keys) == base, f"CF variant {name} differs from the step-by-step split"


def test_fused_operators_match_products():
    """The fast V-cycle's fused level operators (fused.cu) against scipy
    products of the hierarchy's own matrices: A_F P and W_2 = 2Q - Q A_ff Q."""
    import scipy.sparse as sp
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=300, fused_smooths=2)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)

    def csr(m):
        return sp.csr_matrix((m.values, m.col_indices, m.row_offsets), shape=(m.nrows, m.ncols))
    for l in range(h.n_levels):
        A, P, Q, Aff = (csr(h.matrix(l, w)) for w in ("a", "p", "ff_inv", "a_ff"))
        lab = h.labels(l)
        f = np.flatnonzero(lab == 0)
        afp = csr(h.matrix(l, "afp")).toarray()
        np.testing.assert_allclose(afp, (A[f] @ P).toarray(), rtol=1e-13, atol=1e-14 * abs(A).max())
        fw = csr(h.matrix(l, "w")).toarray()
        W = (2 * Q - Q @ Aff @ Q).toarray()
        np.testing.assert_allclose(fw, W, rtol=1e-12, atol=1e-13 * max(1.0, abs(W).max()))


def test_one_pass_operators_match_products():
    """The one-pass ascent's operators against scipy products of the
    hierarchy's own matrices: K = P_F - W_2 A_F P, the descent operator
    [R; W_2 E_F^T], and the composed coarse solve E_3 = Q + E_2 - Q A E_2."""
    import scipy.sparse as sp
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=300, fused_smooths=2)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)

    def csr(m):
        return sp.csr_matrix((m.values, m.col_indices, m.row_offsets), shape=(m.nrows, m.ncols))
    plan = h.fused_plan()
    assert any(plan["one_pass"]) and plan["coarse_composed"]
    for l in range(h.n_levels):
        if not plan["one_pass"][l]:
            continue
        A, P, Q, Aff, R = (csr(h.matrix(l, w)) for w in ("a", "p", "ff_inv", "a_ff", "r"))
        f = np.flatnonzero(h.labels(l) == 0)
        W = 2 * Q - Q @ Aff @ Q
        K = (P[f] - W @ (A[f] @ P)).toarray()
        k = csr(h.matrix(l, "k")).toarray()
        np.testing.assert_allclose(k, K, rtol=1e-12, atol=1e-13 * max(1.0, abs(K).max()))
        EF = sp.csr_matrix((np.ones(len(f)), (np.arange(len(f)), f)), shape=(len(f), A.shape[0]))
        D = sp.vstack([R, W @ EF]).toarray()
        np.testing.assert_allclose(csr(h.matrix(l, "dsc")).toarray(), D, rtol=1e-12,
                                   atol=1e-13 * max(1.0, abs(D).max()))
    L = h.n_levels
    Ac, Qc = csr(h.matrix(L, "a")), csr(h.matrix(L, "ff_inv"))
    E = Qc.copy()
    for _ in range(2):
        E = Qc + E - Qc @ (Ac @ E)
    E = E.toarray()
    np.testing.assert_allclose(csr(h.matrix(L, "coarse_e")).toarray(), E, rtol=1e-11,
                               atol=1e-12 * abs(E).max())


ONE_PASS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
p = problems.make(4, 0.5)
prm = dict(problems.setup_params(4), fused_smooths=2)
h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
v = h.vcycle(p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
g = airg.gmres_solve(h, p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
plan = h.fused_plan()
np.save(sys.argv[1], np.concatenate([v, g.x, [g.stats.iterations, g.stats.final_relative_residual,
        sum(plan["one_pass"]), plan["coarse_composed"]]]))
"""


def test_one_pass_vcycle_matches_two_pass(tmp_path):
    """The fast V-cycle with the one-pass ascent and the composed coarse solve
    equals the two-pass fast V-cycle up to rounding, and the GMRES solve keeps
    its iteration count (+-1) and the 1e-8 solution tolerance."""
    script = tmp_path / "op.py"
    script.write_text(ONE_PASS_SCRIPT % REPO)
    outs = {}
    for name, env in (("one", {"AIRG_ONEPASS_EXTRA": "100000000"}),
                      ("two", {"AIRG_ONEPASS_EXTRA": "-1", "AIRG_COARSE_COMPOSE": "0"})):
        f = tmp_path / f"{name}.npy"
        subprocess.run([sys.executable, str(script), str(f)], check=True, env={**os.environ, **env})
        outs[name] = np.load(f)
    n = (len(outs["one"]) - 4) // 2
    one, two = outs["one"], outs["two"]
    assert one[-2] > 0 and one[-1] == 1 and two[-2] == 0 and two[-1] == 0
    np.testing.assert_allclose(one[:n], two[:n], rtol=0, atol=1e-11 * abs(two[:n]).max())
    assert abs(one[-4] - two[-4]) <= 1 and one[-3] <= 1e-10
    x1, x2 = one[n:2 * n], two[n:2 * n]
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)


@pytest.mark.parametrize("dims", [(9, 9, 9), (7, 5, 3), (8, 8, 6)])
def test_fast_gmres_sweep_shapes(dims):
    """The fast GMRES sweeps take 4 elements per thread when n % 4 == 0, 2
    when n % 4 == 2, and the register-tile kernels when n is odd: every shape
    converges within the parity tolerance of the exact-mode GMRES."""
    nx, ny, nz = dims
    p = problems.c4_tets_3d(nx, ny, nz)
    n_mod = p.n % 4  # 6 tets per cube: n is even; (7, 5, 3) gives n % 4 == 2
    prm = dict(problems.setup_params(4), coarse_size_target=100)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ex = airg.gmres_solve(h, p.b, coarse_iterations=3, max_iterations=300)
    fa = airg.gmres_solve(h, p.b, coarse_iterations=3, max_iterations=300, fast=1)
    assert ex.stats.converged and fa.stats.converged and fa.stats.final_relative_residual <= 1e-10
    assert abs(fa.stats.iterations - ex.stats.iterations) <= 1, (n_mod, fa.stats.iterations, ex.stats.iterations)
    assert np.linalg.norm(fa.x - ex.x) <= 1e-8 * np.linalg.norm(ex.x)


def test_fast_gmres_odd_size():
    """n odd: the fast GMRES falls back to the register-tile sweeps."""
    p = problems.c0_structured_2d(97)
    assert p.n % 2 == 1
    prm = problems.setup_params(0)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    ex = airg.gmres_solve(h, p.b, coarse_iterations=prm["coarse_iterations"], max_iterations=300)
    fa = airg.gmres_solve(h, p.b, coarse_iterations=prm["coarse_iterations"], max_iterations=300, fast=1)
    assert ex.stats.converged and fa.stats.converged and fa.stats.final_relative_residual <= 1e-10
    assert abs(fa.stats.iterations - ex.stats.iterations) <= 1
    assert np.linalg.norm(fa.x - ex.x) <= 1e-8 * np.linalg.norm(ex.x)


COARSE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
p = problems.make(4, 0.25)
prm = dict(problems.setup_params(4), coarse_size_target=300)
h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
out = [h.vcycle(p.b, coarse_iterations=k, fast=1, up_f_smooths=2) for k in (1, 2, 3, 4)]
out.append(h.vcycle(p.b, coarse_iterations=3, fast=1, up_f_smooths=2))  # back to 3: rebuilt, same bits
np.save(sys.argv[1], np.stack(out + [np.full_like(out[0], float(h.fused_plan()["coarse_composed"]))]))
"""


def test_composed_coarse_solve_any_iteration_count(tmp_path):
    """The composed coarse solve E_k (k = 1..4, rebuilt when the solve's
    coarse_iterations changes) equals the k-step coarse Richardson of the
    uncomposed fast V-cycle up to rounding; returning to k = 3 re-captures
    the graphs and reproduces its bits."""
    script = tmp_path / "cs.py"
    script.write_text(COARSE_SCRIPT % REPO)
    outs = {}
    for name, env in (("composed", {}), ("plain", {"AIRG_COARSE_COMPOSE": "0"})):
        f = tmp_path / f"{name}.npy"
        subprocess.run([sys.executable, str(script), str(f)], check=True, env={**os.environ, **env})
        outs[name] = np.load(f)
    a, b = outs["composed"], outs["plain"]
    assert a[-1][0] == 1.0 and b[-1][0] == 0.0
    for k in range(4):
        np.testing.assert_allclose(a[k], b[k], rtol=0, atol=1e-11 * abs(b[k]).max())
    assert np.array_equal(a[2].view(np.uint64), a[4].view(np.uint64))


@pytest.mark.parametrize("nx,ct", [(12, 1000), (40, 700), (64, 300)])
def test_fast_mode_tiny_hierarchies(nx, ct):
    """Coarse-only (no fine level), one-level and two-level hierarchies: the
    fast solve (fused operators, composed coarse solve, one-pass choice,
    device GMRES) matches the exact one to the parity tolerance."""
    p = problems.c0_structured_2d(nx)
    prm = dict(problems.setup_params(0), coarse_size_target=ct)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    if nx == 12:
        assert h.n_levels == 0  # the coarse grid alone
    for outer in (0, 1):
        kw = dict(coarse_iterations=prm["coarse_iterations"], outer=outer, max_iterations=500)
        ex = airg.richardson_solve(h, p.b, **kw)
        fa = airg.richardson_solve(h, p.b, fast=1, **kw)
        assert ex.stats.converged == fa.stats.converged
        if not ex.stats.converged:
            continue
        assert fa.stats.final_relative_residual <= 1e-10
        assert abs(fa.stats.iterations - ex.stats.iterations) <= 1
        assert np.linalg.norm(fa.x - ex.x) <= 1e-8 * np.linalg.norm(ex.x)


def test_fused_rebuild_invalidates_captured_graphs():
    """Switching the F-smooth count rebuilds the fused operators (new
    buffers): every cached graph that captured the old ones must be
    re-captured, so returning to the first count reproduces its bits."""
    p = problems.make(4, 0.25)
    prm = dict(problems.setup_params(4), coarse_size_target=300)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    v2 = h.vcycle(p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
    g2 = airg.gmres_solve(h, p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
    v1 = h.vcycle(p.b, coarse_iterations=3, fast=1, up_f_smooths=1)
    g1 = airg.gmres_solve(h, p.b, coarse_iterations=3, fast=1, up_f_smooths=1)
    assert g1.stats.converged and not np.array_equal(v1, v2)
    v2b = h.vcycle(p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
    g2b = airg.gmres_solve(h, p.b, coarse_iterations=3, fast=1, up_f_smooths=2)
    assert np.array_equal(v2.view(np.uint64), v2b.view(np.uint64))
    assert np.array_equal(g2.x.view(np.uint64), g2b.x.view(np.uint64)) and g2.stats.iterations == g2b.stats.iterations
