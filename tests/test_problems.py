"""Generators for BASELINE.json's five operators (problems.py)."""
import numpy as np
import pytest

from paper_2408_08262_b200 import problems


def _check_csr(p):
    assert p.row_offsets[0] == 0 and p.row_offsets[-1] == len(p.cols) == len(p.vals)
    assert (np.diff(p.row_offsets) >= 0).all()
    for i in range(0, p.n, max(1, p.n // 997)):
        c = p.cols[p.row_offsets[i]:p.row_offsets[i + 1]]
        assert (np.diff(c) > 0).all() and i in c


def test_rng_matches_reference_splitmix():
    # rng.hpp:13-18 known values of splitmix64 (computed by the reference build's formula)
    x = problems.splitmix64(np.array([0, 1, 0xFFFFFFFFFFFFFFFF], np.uint64))
    assert int(x[0]) == 0xE220A8397B1DCDAF
    u = problems.uniform01(np.uint64(7), np.arange(1000, dtype=np.uint64))
    assert (u >= 0).all() and (u < 1).all()


def test_c0_exact_counts():
    p = problems.make(0)
    assert p.n == 16384 and p.nnz == 48896  # SURVEY §8a probe
    _check_csr(p)
    ox, oy = np.cos(0.3), np.sin(0.3)
    assert p.vals[0] == pytest.approx((ox + oy) * 128)


def test_c2_exact_counts():
    p = problems.c2_structured_3d(32)
    assert p.nnz == 4 * p.n - 3 * 32 * 32  # 4n - 3 nx^2
    _check_csr(p)


@pytest.mark.parametrize("cfg,scale", [(1, 0.125), (3, 0.0625), (4, 0.1)])
def test_unstructured_are_upwind_m_matrices(cfg, scale):
    p = problems.make(cfg, scale)
    _check_csr(p)
    d = np.repeat(np.arange(p.n), np.diff(p.row_offsets))
    diag = p.vals[p.cols == d]
    off = p.vals[p.cols != d]
    assert (diag > 0).all() and (off < 0).all()
    # diagonal dominance by columns is what streaming gives; rows: |offdiag| sum <= diag
    rows = np.zeros(p.n)
    np.add.at(rows, d[p.cols != d], np.abs(off))
    assert (rows <= np.abs(diag) * (1 + 1e-12) + 1e-15).all()


def test_generators_deterministic():
    a = problems.make(1, 0.125)
    b = problems.make(1, 0.125)
    assert np.array_equal(a.vals, b.vals) and np.array_equal(a.b, b.b)
