"""One surface over the two implementations under test.

  PortBackend -- the C restatement oracle (oracle/airg_oracle.c, CPU)
  GpuBackend  -- the product: libairg_b200.so through paper_2408_08262_b200.airg

Known-answer tests written once against this surface run on the CPU oracle
in the `not gpu` suite and on the GPU in the `gpu` suite. Matrices are
exchanged as (n, m, rp, ci, v) numpy tuples in the reference layout.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import refpy
from paper_2408_08262_b200 import abi


def triplets(n, m, ts):
    """SparseMatrix::from_triplets (sparse.cpp:48-80) -> (n, m, rp, ci, v)."""
    d = {}
    for r, c, v in ts:
        d[(r, c)] = d.get((r, c), 0.0) + v
    keys = sorted(d)
    rp = np.zeros(n + 1, np.int64)
    for r, _ in keys:
        rp[r + 1] += 1
    return (n, m, np.cumsum(rp), np.array([k[1] for k in keys], np.int64),
            np.array([d[k] for k in keys], np.float64))


def dense(mat):
    n, m, rp, ci, v = mat
    d = np.zeros((n, m))
    for i in range(n):
        d[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return d


def identity(n):
    return (n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))


def diagonal(d):
    n = len(d)
    return (n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.asarray(d, float))


def random_sparse(n, fill, seed, diag_shift=4.0):
    """oracles.hpp:52-68 restated (uniform01 counter stream)."""
    from paper_2408_08262_b200.problems import uniform01
    ctr = np.arange(2 * n * n, dtype=np.uint64)
    u = uniform01(np.uint64(seed), ctr)
    ts = []
    k = 0
    for i in range(n):
        for j in range(n):
            uu, vv = u[k], 2.0 * u[k + 1] - 1.0
            k += 2
            if i == j:
                ts.append((i, j, vv + diag_shift))
            elif uu < fill:
                ts.append((i, j, vv))
    return triplets(n, n, ts)


def random_vector(n, seed):
    from paper_2408_08262_b200.problems import uniform01
    return 2.0 * uniform01(np.uint64(seed), np.arange(n, dtype=np.uint64)) - 1.0


class PortBackend:
    name = "port"
    InvalidArgument = refpy.OracleValueError
    RuntimeErr = refpy.OracleError

    def __init__(self):
        self.lib = refpy.port()

    def _m(self, mat):
        return self.lib.mat(*mat)

    @staticmethod
    def _t(M):
        n, m, _ = M.dims()
        rp, ci, v = M.arrays()
        return (n, m, rp, ci, v)

    def spmv(self, mat, x):
        return refpy.spmv(self.lib, self._m(mat), x)

    def spgemm(self, a, b):
        A, B = self._m(a), self._m(b)
        return self._t(refpy.binop(self.lib, "spgemm", A.h, B.h))

    def drop(self, a, tol, keep=True):
        A = self._m(a)
        return self._t(refpy.binop(self.lib, "drop", A.h, float(tol), int(keep)))

    def full_diag(self, a):
        A = self._m(a)
        return self._t(refpy.binop(self.lib, "with_full_diagonal", A.h))

    def strength(self, a, alpha):
        A = self._m(a)
        out = C.c_void_p()
        st = C.c_int64()
        self.lib.call("strength", A.h, float(alpha), C.byref(out), C.byref(st))
        return self._t(refpy.Mat(self.lib, out, True))

    def pmisr(self, a, alpha, max_loops, seed, mode=0):
        A = self._m(a)
        n = a[0]
        lab = np.zeros(n, np.uint8)
        w = np.zeros(n)
        self.lib.call("pmisr", A.h, float(alpha), int(max_loops), seed, mode, lab, w.ctypes.data_as(C.c_void_p))
        return lab, w

    def pmisr_with_weights(self, s_pattern, max_loops, w):
        S = self._m(s_pattern)
        lab = np.zeros(s_pattern[0], np.uint8)
        self.lib.call("pmisr_with_weights", S.h, int(max_loops), np.ascontiguousarray(w, float), lab)
        return lab

    def cf_split(self, a, seed=0, **kw):
        A = self._m(a)
        lab, pre, rep = refpy.cf_split(self.lib, A, kw, seed)
        return lab, pre, rep

    def ddc(self, a, labels, fraction=0.1, bins=1000, selection=0, direct=0.0):
        A = self._m(a)
        lab = np.ascontiguousarray(labels, np.uint8).copy()
        rep = abi.CfReport()
        self.lib.call("ddc", A.h, lab, float(fraction), int(bins), int(selection), float(direct), C.byref(rep))
        return lab, rep

    def extract(self, a, labels):
        A = self._m(a)
        o = [C.c_void_p(), C.c_void_p(), C.c_void_p()]
        self.lib.call("extract_blocks", A.h, np.ascontiguousarray(labels, np.uint8), *[C.byref(x) for x in o])
        return tuple(self._t(refpy.Mat(self.lib, x, True)) for x in o)

    def coefficients(self, a, m, seed):
        A = self._m(a)
        out = np.zeros(m)
        eff = C.c_int64()
        self.lib.call("poly_coefficients", A.h, int(m), seed, out, C.byref(eff))
        return out, eff.value

    def assemble(self, a, coeffs, eff, s):
        A = self._m(a)
        c = np.ascontiguousarray(coeffs, float)
        return self._t(refpy.binop(self.lib, "poly_assemble", A.h, c, len(c), int(eff), int(s)))

    def setup(self, a, **prm):
        return refpy.setup(self.lib, self._m(a), **prm)

    # single operations (air.hpp:96-116, coarsening.hpp:106, gmres_poly.hpp:40-43, sparse.hpp:133)
    def dominance_report(self, a_ff, bins):
        return refpy.dominance_report(self.lib, self._m(a_ff), bins)

    def label_map(self, labels):
        return refpy.build_label_map(self.lib, labels)

    def restriction(self, a_cf, aff_inv, drop, labels):
        A, B = self._m(a_cf), self._m(aff_inv)
        return self._t(refpy.binop(self.lib, "build_restriction", A.h, B.h, float(drop),
                                   np.ascontiguousarray(labels, np.uint8), len(labels)))

    def prolongation(self, a, s_pattern, labels):
        A, S = self._m(a), self._m(s_pattern)
        return self._t(refpy.binop(self.lib, "build_prolongation", A.h, S.h, np.ascontiguousarray(labels, np.uint8)))

    def coarse_matrix(self, r, a, p, drop):
        R, A, P = self._m(r), self._m(a), self._m(p)
        return self._t(refpy.binop(self.lib, "coarse_matrix", R.h, A.h, P.h, float(drop)))

    def apply_polynomial(self, a, coeffs, eff, b):
        return refpy.apply_polynomial(self.lib, self._m(a), coeffs, eff, b)


class GpuBackend:
    name = "gpu"

    def __init__(self):
        from paper_2408_08262_b200 import airg
        self.airg = airg
        self.InvalidArgument = airg.InvalidArgument
        self.RuntimeErr = airg.AirgRuntimeError

    def _s(self, mat):
        return self.airg.SparseMatrix.from_arrays(*mat)

    @staticmethod
    def _t(S):
        return (S.nrows, S.ncols, S.row_offsets, S.col_indices, S.values)

    def spmv(self, mat, x):
        return self.airg.spmv(self._s(mat), x)

    def spgemm(self, a, b):
        return self._t(self.airg.spgemm(self._s(a), self._s(b)))

    def drop(self, a, tol, keep=True):
        return self._t(self.airg.drop_entries(self._s(a), tol, keep))

    def full_diag(self, a):
        return self._t(self.airg.with_full_diagonal(self._s(a)))

    def strength(self, a, alpha):
        return self._t(self.airg.strength(self._s(a), alpha))

    def pmisr(self, a, alpha, max_loops, seed, mode=0):
        return self.airg.pmisr(self._s(a), alpha, max_loops, seed, mode)

    def pmisr_with_weights(self, s_pattern, max_loops, w):
        return self.airg.pmisr_with_weights(self._s(s_pattern), max_loops, w)

    def cf_split(self, a, seed=0, **kw):
        kw = {**abi.SETUP_DEFAULTS, **kw}
        lab, pre, rep = self.airg.cf_split(self._s(a), kw["strength_alpha"], kw["max_loops"], seed,
                                           kw["weight_mode"], kw["ddc_enabled"], kw["ddc_fraction"],
                                           kw["ddc_bins"])
        return lab, pre, rep

    def ddc(self, a, labels, fraction=0.1, bins=1000, selection=0, direct=0.0):
        return self.airg.ddc(self._s(a), labels, fraction, bins, selection, direct)

    def extract(self, a, labels):
        return tuple(self._t(x) for x in self.airg.extract_blocks(self._s(a), labels))

    def coefficients(self, a, m, seed):
        return self.airg.compute_coefficients(self._s(a), m, seed)

    def assemble(self, a, coeffs, eff, s):
        return self._t(self.airg.assemble_fixed_sparsity(self._s(a), coeffs, eff, s))

    def setup(self, a, **prm):
        return self.airg.setup(self._s(a), **prm)

    def dominance_report(self, a_ff, bins):
        return self.airg.dominance_report(self._s(a_ff), bins)

    def label_map(self, labels):
        return self.airg.build_label_map(labels)

    def restriction(self, a_cf, aff_inv, drop, labels):
        return self._t(self.airg.build_restriction(self._s(a_cf), self._s(aff_inv), drop, labels))

    def prolongation(self, a, s_pattern, labels):
        return self._t(self.airg.build_prolongation(self._s(a), self._s(s_pattern), labels))

    def coarse_matrix(self, r, a, p, drop):
        return self._t(self.airg.coarse_matrix(self._s(r), self._s(a), self._s(p), drop))

    def apply_polynomial(self, a, coeffs, eff, b):
        return self.airg.apply_polynomial(self._s(a), coeffs, eff, b)


def same_bits(x, y) -> bool:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def same_matrix(a, b) -> bool:
    return (a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
            and same_bits(a[4], b[4]))
