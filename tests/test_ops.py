"""The reference's single operations outside the fused setup / solve paths:
dominance_report (coarsening.cpp:219-250), build_label_map (sparse.cpp:
270-290), build_restriction / build_prolongation / coarse_matrix (air.cpp:
154-271), apply_polynomial (gmres_poly.cpp:173-195) and f_smooth
(solve.cpp:63-87).

On the oracle (CPU suite) each is checked against a plain restatement of
its formula; on the GPU (gpu suite) each is bit-identical to the oracle on
the same inputs. oracle/_ref pins the oracle in tests/test_oracle.py.
"""
import numpy as np
import pytest

from backends import GpuBackend, PortBackend, random_sparse, random_vector, same_bits, same_matrix

BACKENDS = [pytest.param("port", id="port"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(scope="module", params=BACKENDS)
def be(request):
    return PortBackend() if request.param == "port" else GpuBackend()


@pytest.fixture(scope="module")
def port():
    return PortBackend()


def _split(port, n, seed):
    """A random operator, its PMISR-DDC labels and blocks (oracle)."""
    a = random_sparse(n, 0.08, seed)
    labels, _, _ = port.cf_split(a, seed=seed)
    aff, afc, acf = port.extract(a, labels)
    return a, labels, aff, afc, acf


def _seq_dot(vals, xs):
    acc = 0.0
    for v, x in zip(vals, xs):
        acc = acc + v * x
    return acc


def _rows(mat):
    n, m, rp, ci, v = mat
    return [(ci[rp[i]:rp[i + 1]], v[rp[i]:rp[i + 1]]) for i in range(n)]


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("bins", [1, 7, 1000])
def test_dominance_report(be, port, seed, bins):
    _, _, aff, _, _ = _split(port, 80, seed)
    theta, hist, mx = be.dominance_report(aff, bins)
    if be.name == "port":
        exp = []
        for i, (c, v) in enumerate(_rows(aff)):
            off = 0.0
            diag = 0.0
            for cc, vv in zip(c, v):
                if cc == i:
                    diag = abs(vv)
                else:
                    off = off + abs(vv)
            exp.append(off / diag)
        exp = np.array(exp)
        assert same_bits(theta, exp)
        assert mx == exp.max()
        width = mx / bins if mx > 0 else 1.0
        eh = np.zeros(bins, np.int64)
        for t in exp:
            eh[min(int(t / width), bins - 1)] += 1
        assert np.array_equal(hist, eh)
    else:
        t2, h2, m2 = port.dominance_report(aff, bins)
        assert same_bits(theta, t2) and np.array_equal(hist, h2) and m2 == mx


def test_dominance_report_zero_diagonal(be):  # coarsening.cpp:237-239
    a = (2, 2, np.array([0, 1, 2]), np.array([1, 1]), np.array([1.0, 2.0]))  # row 0 lacks its diagonal
    with pytest.raises(be.RuntimeErr, match="zero diagonal in A_ff row 0"):
        be.dominance_report(a, 10)
    with pytest.raises(be.InvalidArgument):
        be.dominance_report(a, 0)


@pytest.mark.parametrize("seed", [0, 5])
def test_label_map(be, seed):
    lab = (np.random.default_rng(seed).random(57) < 0.4).astype(np.uint8)  # F = 0, C = 1
    f2s, f2f, c2f = be.label_map(lab)
    assert np.array_equal(f2f, np.flatnonzero(lab == 0))
    assert np.array_equal(c2f, np.flatnonzero(lab == 1))
    exp = np.empty(len(lab), np.int64)
    exp[f2f] = np.arange(len(f2f))
    exp[c2f] = np.arange(len(c2f))
    assert np.array_equal(f2s, exp)


@pytest.mark.parametrize("seed", [1, 4])
def test_transfer_operators(be, port, seed):
    a, labels, aff, afc, acf = _split(port, 90, seed)
    coeffs, eff = port.coefficients(aff, 3, seed)
    ffinv = port.assemble(aff, coeffs, eff, 1)
    r = be.restriction(acf, ffinv, 0.01, labels)
    s = port.strength(a, 0.5)
    p = be.prolongation(a, s, labels)
    ac = be.coarse_matrix(r, a, p, 0.001)
    if be.name == "port":
        nc = int(np.count_nonzero(labels == 1))
        c2f = np.flatnonzero(labels == 1)
        # R's C columns carry the identity (air.cpp:179-184)
        for c, (cols, vals) in enumerate(_rows(r)):
            k = list(cols).index(c2f[c])
            assert vals[k] == 1.0
        # one-point P: C rows are identity rows, F rows at most one 1.0
        rows = _rows(p)
        for i in range(a[0]):
            cols, vals = rows[i]
            assert len(cols) <= 1 and all(v == 1.0 for v in vals)
            if labels[i] == 1:
                assert len(cols) == 1
        assert ac[0] == ac[1] == nc
    else:
        assert same_matrix(r, port.restriction(acf, ffinv, 0.01, labels))
        assert same_matrix(p, port.prolongation(a, s, labels))
        assert same_matrix(ac, port.coarse_matrix(r, a, p, 0.001))


@pytest.mark.parametrize("seed", [2, 3])
@pytest.mark.parametrize("m", [1, 3, 6])
def test_apply_polynomial(be, port, seed, m):
    a = random_sparse(70, 0.07, 100 + seed)
    b = random_vector(70, seed)
    coeffs, eff = port.coefficients(a, m, seed)
    y = be.apply_polynomial(a, coeffs, eff, b)
    if be.name == "port":
        rows = _rows(a)
        acc = [coeffs[eff] * bi for bi in b]
        for k in range(eff - 1, -1, -1):
            t = [_seq_dot(v, [acc[j] for j in c]) for c, v in rows]
            acc = [ti + coeffs[k] * bi for ti, bi in zip(t, b)]
        assert same_bits(y, np.array(acc))
    else:
        assert same_bits(y, port.apply_polynomial(a, coeffs, eff, b))


def test_apply_polynomial_errors(be):
    a = random_sparse(10, 0.3, 9)
    with pytest.raises(be.InvalidArgument):
        be.apply_polynomial(a, [], 0, np.ones(10))


def test_f_smooth(be):
    """One F-smooth on level 0 of a built hierarchy equals the reference's
    composition (solve.cpp:63-87) over that hierarchy's own level matrices."""
    from paper_2408_08262_b200 import problems
    p = problems.c2_structured_3d(12)
    a = (p.n, p.n, p.row_offsets, p.cols, p.vals)
    prm = dict(problems.setup_params(2), coarse_size_target=200)
    h = be.setup(a, **prm)
    labels = h.labels(0)
    if be.name == "port":
        mats = [(m.dims()[0], m.dims()[1], *m.arrays()) for m in (h.matrix(0, w) for w in (1, 2, 4))]
    else:
        mats = []
        for w in ("a_ff", "a_fc", "ff_inv"):
            s = h.matrix(0, w)
            mats.append((s.nrows, s.ncols, s.row_offsets, s.col_indices, s.values))
    aff, afc, ffinv = mats
    f2f = np.flatnonzero(labels == 0)
    c2f = np.flatnonzero(labels == 1)
    b = random_vector(p.n, 3)
    x = random_vector(p.n, 4)
    got = h.f_smooth(0, b, x)
    port = PortBackend()
    rf = port.spmv(aff, x[f2f])
    sc = port.spmv(afc, x[c2f])
    r = np.array([(b[f] - rf[k]) - sc[k] for k, f in enumerate(f2f)])
    d = port.spmv(ffinv, r)
    exp = x.copy()
    exp[f2f] = exp[f2f] + d
    assert same_bits(got, exp)
    assert same_bits(got[c2f], x[c2f])


@pytest.mark.gpu
def test_device_buffer_helpers_round_trip():
    """airg_device_alloc / airg_memcpy / airg_device_free (the buffers the
    C++ adapter uses without linking CUDA)."""
    import ctypes as C
    from paper_2408_08262_b200 import airg
    L = airg.lib()
    for name, args in (("airg_device_alloc", [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
                       ("airg_device_free", [C.c_void_p, C.c_void_p]),
                       ("airg_memcpy", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32])):
        getattr(L, name).argtypes = args
        getattr(L, name).restype = C.c_int
    ctx = airg.default_context()
    src = np.random.default_rng(0).random(1000)
    dst = np.zeros_like(src)
    p = C.c_void_p()
    assert L.airg_device_alloc(ctx.h, src.nbytes, C.byref(p)) == 0 and p.value
    assert L.airg_memcpy(ctx.h, p, src.ctypes.data, src.nbytes, 1) == 0
    assert L.airg_memcpy(ctx.h, dst.ctypes.data, p, src.nbytes, 0) == 0
    assert L.airg_device_free(ctx.h, p) == 0
    assert same_bits(src, dst)



@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 8192, 135169, 3 * 4096 * 40 + 5, 6_000_001])
@pytest.mark.parametrize("frac_f", [0.0, 0.37, 1.0])
def test_label_map_sizes_across_scan_tiles(n, frac_f):
    """The label map's F/C positions come from the single-pass look-back scan
    (util.cu scan_lookback: 4096-element tiles, 32-tile look-back windows):
    one element, tile boundaries, several look-back windows (> 32 tiles), all
    F / all C / mixed -- against the numpy positions (sparse.cpp:270-290)."""
    from paper_2408_08262_b200 import airg
    rng = np.random.default_rng(n)
    lab = (rng.random(n) >= frac_f).astype(np.uint8)  # 0 = F, 1 = C
    f2s, f2f, c2f = airg.build_label_map(lab)
    isf = lab == 0
    assert np.array_equal(f2f, np.flatnonzero(isf))
    assert np.array_equal(c2f, np.flatnonzero(~isf))
    want = np.where(isf, np.cumsum(isf) - 1, np.cumsum(~isf) - 1)
    assert np.array_equal(f2s, want)


_CF_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, %r)
sys.path.insert(0, %r)
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
from backends import PortBackend
port = PortBackend()
for nx in (12, 20):
    p = problems.c2_structured_3d(nx)
    a = (p.n, p.n, p.row_offsets, p.cols, p.vals)
    for seed in (0, 3):
        lab, pre, rep = airg.cf_split(airg.SparseMatrix.from_arrays(*a), 0.5, 3, seed)
        exp, exp_pre, _ = port.cf_split(a, seed=seed)
        assert np.array_equal(lab, exp) and np.array_equal(pre, exp_pre), (nx, seed)
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"AIRG_CF_VEC": "1"}, {"AIRG_CF_VEC": "100000"}, {"AIRG_PDL": "0"}],
                         ids=["default", "vector_rows", "scalar_rows", "no_pdl"])
def test_fused_cf_split_schedules_match_oracle(env):
    """The fused split with 16-byte / scalar row loads and without PDL (read
    once per process, hence a subprocess each) gives the oracle's labels bit
    for bit."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _CF_SCRIPT % (repo, os.path.join(repo, "tests"), os.path.join(repo, "oracle"))
    full = dict(os.environ)
    full.update(env)
    out = subprocess.run([sys.executable, "-c", script], env=full, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


_SETUP_SCRIPT = r"""
import hashlib
import sys
import numpy as np
sys.path.insert(0, %r)
from paper_2408_08262_b200 import airg, problems
dg = hashlib.sha256()
for cfg, scale in ((4, 0.5), (2, 0.25)):
    p = problems.make(cfg, scale)
    prm = dict(problems.setup_params(cfg), fused_smooths=2)
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    retried = 0
    for l in range(h.n_levels):
        L = h.level(l)
        retried += L.smoother_growth > 0.5 or L.poly_attempts > 1
        dg.update(h.labels(l).tobytes())
        dg.update(np.array([L.poly_attempts, L.effective_order], np.int64).tobytes())
        dg.update(np.array([L.smoother_growth], np.float64).tobytes())
        for which in ("a", "ff_inv", "r", "p", "afp", "w"):
            m = h.matrix(l, which)
            for arr in (m.row_offsets, m.col_indices, m.values):
                dg.update(np.ascontiguousarray(arr).tobytes())
    res = airg.gmres_solve(h, p.b, coarse_iterations=prm["coarse_iterations"], fast=1)
    dg.update(res.x.tobytes())
    print("retried", cfg, int(retried))
print("digest", dg.hexdigest())
"""


@pytest.mark.gpu
def test_side_by_side_setup_chains_same_hierarchy():
    """AIRG_SETUP_PARALLEL (setup.cu / fused.cu: the retry fits, the fused
    operators, P and A P enqueued by host threads on worker streams) changes
    the schedule only: labels, attempts, growth, level operators, fused
    operators and the fast solve are bit-identical for masks 0, 1 and 7 (the
    mask is read once per process, hence subprocesses). The half-size C4
    hierarchy has levels whose first fit fails the growth guard."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mask in ("0", "1", "7"):
        env = dict(os.environ, AIRG_SETUP_PARALLEL=mask)
        out = subprocess.run([sys.executable, "-c", _SETUP_SCRIPT % repo], env=env, capture_output=True, text=True,
                             timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        outs[mask] = out.stdout.strip().splitlines()
    assert outs["0"][-1].startswith("digest ")
    assert outs["0"] == outs["1"] == outs["7"], outs
    assert any(ln.startswith("retried 4 ") and int(ln.split()[-1]) > 0 for ln in outs["0"]), outs["0"]
