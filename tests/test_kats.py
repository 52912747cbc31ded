"""The reference's own known-answer tests, restated once and run against both
implementations: the C oracle (CPU suite) and the GPU engine (gpu suite).

Each test cites the reference test it restates (proj/tests/unit/*.cpp).
"""
import numpy as np
import pytest

from backends import (GpuBackend, PortBackend, dense, diagonal, identity, random_sparse,
                      random_vector, same_bits, same_matrix, triplets)

BACKENDS = [pytest.param("port", id="port"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(scope="module", params=BACKENDS)
def be(request):
    return PortBackend() if request.param == "port" else GpuBackend()


# ---- sparse kernels (test_sparse.cpp) -------------------------------------------
def test_spmv_identity_and_diagonal(be):  # test_sparse.cpp:12-21
    assert np.array_equal(be.spmv(identity(3), [1, 2, 3]), [1, 2, 3])
    assert np.array_equal(be.spmv(diagonal([2, 3]), [1, 1]), [2, 3])


def test_spmv_matches_dense(be):  # test_sparse.cpp:23-31
    a = random_sparse(5, 0.6, 11)
    x = random_vector(5, 7)
    np.testing.assert_allclose(be.spmv(a, x), dense(a) @ x, rtol=1e-14, atol=1e-14)


def test_spmv_dimension_check(be):  # test_sparse.cpp:33-39
    a = random_sparse(8, 0.4, 3)
    with pytest.raises(ValueError):
        be.spmv(a, np.ones(7))


def test_spgemm_small_cases(be):  # test_sparse.cpp:41-51
    a = triplets(2, 2, [(0, 0, 1), (0, 1, 1), (1, 1, 1)])
    assert same_matrix(be.spgemm(a, identity(2)), a)
    b = triplets(2, 2, [(0, 0, 1), (1, 0, 1), (1, 1, 1)])
    assert np.array_equal(dense(be.spgemm(a, b)), [[2, 1], [1, 1]])


def test_spgemm_keeps_cancellation_zeros(be):  # test_sparse.cpp:72-79
    a = triplets(1, 2, [(0, 0, 1), (0, 1, 1)])
    b = triplets(2, 1, [(0, 0, 1), (1, 0, -1)])
    c = be.spgemm(a, b)
    assert c[2][-1] == 1 and c[4][0] == 0.0


def test_spgemm_rectangular_and_associative(be):  # test_sparse.cpp:53-70, :81-90
    for s in range(6):
        r, a, p = (random_sparse(9, 0.3, 100 + s), random_sparse(9, 0.3, 200 + s),
                   random_sparse(9, 0.3, 300 + s))
        left = be.spgemm(be.spgemm(r, a), p)
        right = be.spgemm(r, be.spgemm(a, p))
        assert np.abs(dense(left) - dense(right)).max() < 1e-12
    with pytest.raises(ValueError):
        be.spgemm(triplets(2, 3, [(0, 0, 1.0)]), triplets(2, 3, [(0, 0, 1.0)]))


def test_drop_rules(be):  # test_sparse.cpp:154-187
    a = random_sparse(7, 0.5, 9)
    assert same_matrix(be.drop(a, 0.0), a)
    row = triplets(1, 3, [(0, 0, 4.0), (0, 1, 0.01), (0, 2, 1.0)])
    assert list(be.drop(row, 0.1)[3]) == [0, 2]
    tiny = triplets(2, 2, [(0, 0, 1e-20), (0, 1, 5.0), (1, 1, 1.0)])
    assert 0 in list(be.drop(tiny, 0.9)[3][:be.drop(tiny, 0.9)[2][1]])
    z = triplets(2, 3, [(0, 0, 0.5), (0, 2, -2.0), (1, 1, 0.1), (1, 2, 0.099)])
    d = be.drop(z, 1.1)
    assert d[2][-1] == 2 and list(d[4]) == [-2.0, 0.1]
    for tol in (0.05, 0.3, 1.5):
        once = be.drop(random_sparse(10, 0.5, 77), tol)
        assert same_matrix(be.drop(once, tol), once)
    with pytest.raises(ValueError):
        be.drop(a, -1.0)


def test_with_full_diagonal(be):  # test_sparse.cpp:189-198
    a = triplets(3, 3, [(0, 1, 2.0), (2, 2, 1.0)])
    full = be.full_diag(a)
    assert full[2][-1] == 4
    assert np.array_equal(dense(full), [[0, 2, 0], [0, 0, 0], [0, 0, 1]])
    assert same_matrix(be.full_diag(full), full)


def test_extract_blocks_round_trip(be):  # test_sparse.cpp:92-146
    from paper_2408_08262_b200.problems import uniform01
    for s in range(4):
        a = random_sparse(12, 0.4, 50 + s)
        labels = (uniform01(np.uint64(s), np.arange(12, dtype=np.uint64)) >= 0.5).astype(np.uint8)
        aff, afc, acf = be.extract(a, labels)
        d = dense(a)
        f = np.where(labels == 0)[0]
        c = np.where(labels == 1)[0]
        assert np.array_equal(dense(aff), d[np.ix_(f, f)])
        assert np.array_equal(dense(afc), d[np.ix_(f, c)])
        assert np.array_equal(dense(acf), d[np.ix_(c, f)])
    with pytest.raises(ValueError):
        be.extract(identity(2), [0, 2])


# ---- strength / PMISR / DDC (test_coarsening.cpp) -----------------------------------
def test_strength_identity_empty(be):  # test_coarsening.cpp:30-34
    assert be.strength(identity(5), 0.3)[2][-1] == 0


def test_strength_tridiagonal(be):  # test_coarsening.cpp:36-50
    n = 6
    ts = []
    for i in range(n):
        ts.append((i, i, 2.0))
        if i > 0:
            ts.append((i, i - 1, -1.0))
        if i + 1 < n:
            ts.append((i, i + 1, -1.0))
    s = be.strength(triplets(n, n, ts), 0.5)
    assert list(np.diff(s[2])) == [1, 2, 2, 2, 2, 1]


def test_strength_threshold_within_row(be):  # test_coarsening.cpp:52-66
    s = be.strength(triplets(2, 2, [(0, 0, 1), (0, 1, 4), (1, 0, 0.1), (1, 1, 1)]), 0.5)
    assert list(np.diff(s[2])) == [1, 1]
    s = be.strength(triplets(3, 3, [(0, 0, 1), (0, 1, 4), (0, 2, 0.1), (1, 1, 1), (2, 2, 1)]), 0.5)
    assert list(s[3][s[2][0]:s[2][1]]) == [1]


def test_strength_alpha_zero_is_adjacency(be):  # test_coarsening.cpp:68-84
    a = random_sparse(15, 0.3, 42)
    s = be.strength(a, 0.0)
    n, _, rp, ci, v = a
    for i in range(15):
        exp = {ci[k] for k in range(rp[i], rp[i + 1]) if ci[k] != i and v[k] != 0.0}
        assert set(s[3][s[2][i]:s[2][i + 1]]) == exp
    z = triplets(2, 2, [(0, 0, 1.0), (0, 1, 0.0), (1, 1, 1.0)])
    assert be.strength(z, 0.0)[2][1] == 0


def test_pmisr_empty_graph_all_f(be):  # test_coarsening.cpp:91-96
    lab, w = be.pmisr(identity(8), 0.5, 3, 1)
    assert (lab == 0).all() and (w < 1.0).all()


def test_pmisr_pair_and_k3(be):  # test_coarsening.cpp:98-122
    pair = triplets(2, 2, [(0, 1, 1.0), (1, 0, 1.0)])
    for w in ([2.3, 2.7], [2.7, 2.3]):
        lab = be.pmisr_with_weights(pair, 3, w)
        f = 0 if w[0] < w[1] else 1
        assert lab[f] == 0 and lab[1 - f] == 1
    k3 = triplets(3, 3, [(0, 1, 1), (0, 2, 1), (1, 0, 1), (1, 2, 1), (2, 0, 1), (2, 1, 1)])
    for w in ([4.1, 4.5, 4.9], [4.1, 4.9, 4.5], [4.5, 4.1, 4.9], [4.9, 4.1, 4.5], [4.5, 4.9, 4.1],
              [4.9, 4.5, 4.1]):
        lab = be.pmisr_with_weights(k3, 3, w)
        assert (lab == 0).sum() == 1 and lab[int(np.argmin(w))] == 0


def _independent(s, lab):
    n, _, rp, ci, _ = s
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            if lab[i] == 0 and lab[ci[k]] == 0:
                return False
    return True


def test_pmisr_independent_random(be):  # test_coarsening.cpp:124-132
    for s in range(25):
        a = random_sparse(60, 0.08, 900 + s)
        lab, _ = be.pmisr(a, 0.25, 3, s)
        assert _independent(be.strength(a, 0.25), lab)
        assert set(np.unique(lab)) <= {0, 1}


def test_pmisr_deterministic_and_capped(be):  # test_coarsening.cpp:134-147
    a = random_sparse(80, 0.1, 31)
    l1, w1 = be.pmisr(a, 0.4, 3, 7)
    l2, w2 = be.pmisr(a, 0.4, 3, 7)
    assert np.array_equal(l1, l2) and same_bits(w1, w2)
    capped, _ = be.pmisr(a, 0.4, 1, 7)
    uncapped, _ = be.pmisr(a, 0.4, 1000, 7)
    assert set(np.where(capped == 0)[0]) <= set(np.where(uncapped == 0)[0])
    with pytest.raises(ValueError):
        be.pmisr(a, 0.4, 0, 7)


def test_pmisr_weight_modes(be):  # test_coarsening.cpp:149-157
    g = triplets(3, 3, [(0, 1, 1.0), (1, 0, 1.0), (1, 2, 1.0), (2, 1, 1.0)])
    _, ws = be.pmisr(g, 0.5, 3, 5, 0)
    _, wu = be.pmisr(g, 0.5, 3, 5, 1)
    assert ws[1] > 4.0 and wu[1] < 3.0 and abs((ws[1] - wu[1]) - 2.0) < 1e-12


def test_alpha_zero_gives_diagonal_aff(be):  # test_coarsening.cpp:159-167
    for s in range(5):
        a = random_sparse(40, 0.15, 700 + s)
        lab, _ = be.pmisr(a, 0.0, 3, s)
        aff, _, _ = be.extract(a, lab)
        n, _, rp, ci, _ = aff
        assert all(ci[k] == i for i in range(n) for k in range(rp[i], rp[i + 1]))


def test_ddc_diagonal_untouched(be):  # test_coarsening.cpp:207-222
    for frac in (0.1, 0.5, 1.0):
        lab, rep = be.ddc(diagonal([1.0, 2.0, 3.0]), [0, 0, 0], fraction=frac)
        assert rep.n_converted == 0 and list(lab) == [0, 0, 0]


def test_ddc_direct_converts_dominated_row(be):  # test_coarsening.cpp:224-239
    a = triplets(2, 2, [(0, 0, 1.0), (0, 1, 2.0), (1, 1, 1.0)])
    lab, rep = be.ddc(a, [0, 0], selection=2, direct=1.0)
    assert list(lab) == [1, 0] and rep.n_converted == 1


def test_ddc_histogram_within_one(be):  # test_coarsening.cpp:241-270
    n = 100
    ts = [(i, i, 1.0) for i in range(n)] + [(i, (i + 1) % n, 0.01 * (i + 1)) for i in range(n)]
    lab, rep = be.ddc(triplets(n, n, ts), np.zeros(n, np.uint8), fraction=0.10, bins=1000)
    assert 9 <= rep.n_converted <= 11


def test_ddc_quickselect_exact(be):  # test_coarsening.cpp:241-263 (kQuickSelect)
    n = 100
    ts = [(i, i, 1.0) for i in range(n)] + [(i, (i + 1) % n, 0.01 * (i + 1)) for i in range(n)]
    lab, rep = be.ddc(triplets(n, n, ts), np.zeros(n, np.uint8), fraction=0.10, selection=1)
    assert rep.n_converted == 10 and (np.flatnonzero(lab) >= 90).all() and lab.sum() == 10


def test_ddc_quickselect_edges_and_random(be):  # coarsening.cpp:270-288 edge cases
    for frac in (0.001, 0.999, 1.0):  # target 0, n_f, n_f
        n = 50
        ts = [(i, i, 1.0) for i in range(n)] + [(i, (i + 3) % n, 0.02 * ((7 * i) % n + 1)) for i in range(n)]
        lab, rep = be.ddc(triplets(n, n, ts), np.zeros(n, np.uint8), fraction=frac, selection=1)
        want = 0 if frac < 0.01 else n
        assert rep.n_converted == want, (frac, rep.n_converted)
    for s in range(4):  # random magnitudes: the exact order statistic's conversions
        a = be.full_diag(random_sparse(60, 0.1, 900 + s))
        n, _, rp, ci, v = a
        theta = []
        for i in range(n):
            off, dg = 0.0, 0.0
            for k in range(rp[i], rp[i + 1]):
                if ci[k] == i:
                    dg = abs(v[k])
                else:
                    off += abs(v[k])
            theta.append(off / dg)
        theta = np.array(theta)
        target = int(np.round(0.25 * n))
        alpha = np.sort(theta)[n - target - 1]
        want = np.flatnonzero((theta > alpha) & (theta != 0))
        lab, rep = be.ddc(a, np.zeros(n, np.uint8), fraction=0.25, selection=1)
        assert np.array_equal(np.flatnonzero(lab), want), s


def test_ddc_measures_theta_once(be):  # test_coarsening.cpp:272-289
    a = triplets(3, 3, [(0, 0, 1.0), (0, 1, 3.0), (1, 0, 3.0), (1, 1, 1.0), (2, 2, 1.0)])
    lab, rep = be.ddc(a, [0, 0, 0], selection=2, direct=2.0)
    assert rep.n_converted == 2 and lab[2] == 0


def test_ddc_zero_diagonal_names_row(be):  # test_coarsening.cpp:291-301
    a = be.full_diag(triplets(2, 2, [(0, 0, 1.0), (1, 0, 1.0)]))
    with pytest.raises(RuntimeError, match="row 1"):
        be.ddc(a, [0, 0])


# ---- polynomials (test_gmres_poly.cpp) -----------------------------------------------
def test_identity_collapses_to_one(be):  # test_gmres_poly.cpp:24-33
    for m in (1, 3, 7):
        c, eff = be.coefficients(identity(10), m, 4)
        assert eff == 0 and abs(c[0] - 1.0) < 1e-12 and (c[1:] == 0).all()


def test_scaled_identity(be):  # test_gmres_poly.cpp:35-40
    c, eff = be.coefficients(diagonal([2.0] * 6), 3, 9)
    assert eff == 0 and abs(c[0] - 0.5) < 1e-12


def test_two_eigenvalues(be):  # test_gmres_poly.cpp:42-54
    c, _ = be.coefficients(diagonal([1.0, 2.0]), 2, 17)
    assert abs(c[0] - 1.5) < 1e-10 and abs(c[1] + 0.5) < 1e-10


def test_k_distinct_eigenvalues(be):  # test_gmres_poly.cpp:82-95
    for k in range(1, 9):
        n = 40
        d = [3.0] * n if k == 1 else [1.0 + 9.0 * (i % k) / max(1, k - 1) for i in range(n)]
        c, eff = be.coefficients(diagonal(d), k + 1, 23 + k)
        b = random_vector(n, 99 + k)
        x = np.zeros(n)
        dd = np.array(d)
        for j in range(eff, -1, -1):  # Horner, apply_polynomial (gmres_poly.cpp:173-195)
            x = dd * x + c[j] * b
        assert np.linalg.norm(b - dd * x) / np.linalg.norm(b) < 1e-8


def test_assembled_diagonal_closure(be):  # test_gmres_poly.cpp:97-113
    d = [1.0, 2.5, 4.0, 8.0]
    c, eff = be.coefficients(diagonal(d), 4, 6)
    for s in (1, 3):
        inv = be.assemble(diagonal(d), c, eff, s)
        assert list(inv[3]) == [0, 1, 2, 3]
        for i in range(4):
            q = sum(c[k] * d[i] ** k for k in range(len(c)))
            assert abs(inv[4][i] - q) <= 1e-12 * max(1.0, abs(q))


def test_fixed_sparsity_matches_dense_oracle(be):  # test_gmres_poly.cpp:129-147
    n = 8
    ts = []
    for i in range(n):
        ts.append((i, i, 3.0 + 0.1 * i))
        if i > 0:
            ts.append((i, i - 1, -1.0))
        if i + 1 < n:
            ts.append((i, i + 1, -1.2))
    a = triplets(n, n, ts)
    c, eff = be.coefficients(a, 4, 15)
    inv = be.assemble(a, c, eff, 1)
    ad = dense(a)
    mask = (ad != 0) | np.eye(n, dtype=bool)
    res = c[0] * np.eye(n) + (c[1] * ad if eff >= 1 else 0)
    p = ad.copy()
    for k in range(2, eff + 1):
        p = (p @ ad) * mask
        res = res + c[k] * p
    assert np.abs(dense(inv) - res).max() < 1e-13


def test_coefficient_argument_validation(be):  # test_gmres_poly.cpp:179-184
    with pytest.raises(ValueError):
        be.coefficients(identity(3), 0, 1)
    with pytest.raises(ValueError):
        be.coefficients(triplets(2, 3, [(0, 0, 1.0)]), 2, 1)
