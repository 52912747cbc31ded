"""Python mirror of the reference's airgraph:: API over the B200 C-ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/airgraph/*.hpp (cited per function) so the
parity tests read like the reference's own tests:
  std::invalid_argument -> InvalidArgument (a ValueError)
  std::runtime_error    -> AirgRuntimeError (a RuntimeError)
Every compute call goes through paper_2408_08262_b200/libairg_b200.so
(hand-written sm_100a kernels); there is no CPU fallback: if the library is
missing or no CUDA device is present, the calls raise.

Device memory and streams come from PyTorch (plumbing only): the context
runs its kernels on a dedicated torch stream whose handle is handed to the
C-ABI, and device tensors are passed as raw pointers.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# AIRG_LIB: an alternative build of the same engine (A/B variants built by
# `make -C csrc variant V=<tag> XFLAGS=...`, tools/ab_variants.sh); default in-tree
LIB_PATH = os.environ.get("AIRG_LIB") or os.path.join(HERE, "libairg_b200.so")


class InvalidArgument(ValueError):
    """std::invalid_argument at the reference boundary."""


class AirgRuntimeError(RuntimeError):
    """std::runtime_error at the reference boundary (stall, zero diagonal)."""


class CudaFailure(RuntimeError):
    pass


_lib = None
_VP = C.c_void_p
_P = C.POINTER


def lib() -> C.CDLL:
    """Load the CUDA engine; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a engine first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        sig = {
            "airg_last_error": ([C.c_char_p, C.c_size_t], C.c_int),
            "airg_version": ([], C.c_char_p),
            "airg_setup_config_default": ([_P(abi.SetupConfig)], None),
            "airg_solve_config_default": ([_P(abi.SolveConfig)], None),
            "airg_ctx_create": ([C.c_int, _P(_VP)], C.c_int),
            "airg_ctx_destroy": ([_VP], C.c_int),
            "airg_ctx_set_stream": ([_VP, _VP], C.c_int),
            "airg_ctx_synchronize": ([_VP], C.c_int),
            "airg_ctx_launch_count": ([_VP, _P(C.c_uint64)], C.c_int),
            "airg_csr_upload": ([_VP, C.c_int64, C.c_int64, _VP, _VP, _VP, _P(_VP)], C.c_int),
            "airg_csr_info": ([_VP, _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)], C.c_int),
            "airg_csr_download": ([_VP, _VP, _VP, _VP, _VP], C.c_int),
            "airg_csr_device_ptrs": ([_VP, _P(_VP), _P(_VP), _P(_VP)], C.c_int),
            "airg_csr_destroy": ([_VP], C.c_int),
            "airg_spmv": ([_VP, _VP, _VP, _VP], C.c_int),
            "airg_spgemm": ([_VP, _VP, _VP, _P(_VP)], C.c_int),
            "airg_drop": ([_VP, _VP, C.c_double, C.c_int, _P(_VP)], C.c_int),
            "airg_with_full_diagonal": ([_VP, _VP, _P(_VP)], C.c_int),
            "airg_strength": ([_VP, _VP, C.c_double, _P(_VP)], C.c_int),
            "airg_pmisr": ([_VP, _VP, C.c_double, C.c_int64, C.c_uint64, C.c_int32, _VP, _VP], C.c_int),
            "airg_pmisr_with_weights": ([_VP, _VP, C.c_int64, _VP, _VP], C.c_int),
            "airg_pmis": ([_VP, _VP, C.c_double, C.c_int32, C.c_uint64, _VP], C.c_int),
            "airg_cf_split": ([_VP, _VP, C.c_double, C.c_int64, C.c_uint64, C.c_int32, C.c_int32,
                               C.c_double, C.c_int64, _VP, _VP, _P(abi.CfReport)], C.c_int),
            "airg_cf_split_batch": ([_VP, _VP, C.c_int64, _VP, C.c_double, C.c_int64, C.c_int32,
                                     C.c_double, C.c_int64, _VP, _P(abi.CfReport)], C.c_int),
            "airg_ddc": ([_VP, _VP, _VP, C.c_double, C.c_int64, C.c_int32, C.c_double,
                          _P(abi.CfReport)], C.c_int),
            "airg_extract_blocks": ([_VP, _VP, _VP, _P(_VP), _P(_VP), _P(_VP)], C.c_int),
            "airg_poly_coefficients": ([_VP, _VP, C.c_int64, C.c_uint64, _VP, _P(C.c_int64)], C.c_int),
            "airg_poly_assemble": ([_VP, _VP, _VP, C.c_int64, C.c_int64, C.c_int64, _P(_VP)], C.c_int),
            "airg_setup": ([_VP, _VP, _P(abi.SetupConfig), _P(abi.Injection), _P(_VP)], C.c_int),
            "airg_dist_setup": ([_VP, _VP, _P(abi.SetupConfig), _P(abi.Injection), C.c_int32, C.c_int32, _VP,
                                 _P(_VP)], C.c_int),
            "airg_hier_info_get": ([_VP, _P(abi.HierInfo)], C.c_int),
            "airg_hier_level_info": ([_VP, C.c_int64, _P(abi.LevelInfo)], C.c_int),
            "airg_hier_matrix": ([_VP, C.c_int64, C.c_int32, _P(_VP)], C.c_int),
            "airg_hier_labels": ([_VP, _VP, C.c_int64, _VP], C.c_int),
            "airg_hier_destroy": ([_VP], C.c_int),
            "airg_vcycle": ([_VP, _VP, _P(abi.SolveConfig), _VP, _VP], C.c_int),
            "airg_f_smooth": ([_VP, _VP, C.c_int64, _VP, _VP], C.c_int),
            "airg_dominance_report": ([_VP, _VP, C.c_int64, _VP, _VP, _P(C.c_double)], C.c_int),
            "airg_build_label_map": ([_VP, _VP, C.c_int64, _VP, _VP, _VP, _P(C.c_int64)], C.c_int),
            "airg_build_restriction": ([_VP, _VP, _VP, C.c_double, _VP, C.c_int64, _P(_VP)], C.c_int),
            "airg_build_prolongation": ([_VP, _VP, _VP, _VP, _P(_VP)], C.c_int),
            "airg_coarse_matrix": ([_VP, _VP, _VP, _VP, C.c_double, _P(_VP)], C.c_int),
            "airg_apply_polynomial": ([_VP, _VP, _VP, C.c_int64, C.c_int64, _VP, _VP], C.c_int),
            "airg_solve": ([_VP, _VP, _P(abi.SolveConfig), _VP, _VP, _P(abi.SolveStats), _VP,
                            C.c_int64], C.c_int),
            "airg_solve_host": ([_VP, _VP, _P(abi.SolveConfig), _VP, _VP, _P(abi.SolveStats), _VP,
                                 C.c_int64], C.c_int),
            "airg_spmv_host": ([_VP, _VP, _VP, _VP], C.c_int),
            "airg_cf_split_host": ([_VP, _VP, C.c_double, C.c_int64, C.c_uint64, C.c_int32, C.c_int32,
                                    C.c_double, C.c_int64, _VP, _P(abi.CfReport)], C.c_int),
            "airg_nccl_unique_id": ([_VP], C.c_int),
            "airg_nccl_comm_create": ([C.c_int, C.c_int, _VP, _P(_VP)], C.c_int),
            "airg_nccl_comm_destroy": ([_VP], C.c_int),
            "airg_dist_setup_owned": ([_VP, _VP, _VP, _P(abi.SetupConfig), _P(abi.Injection), C.c_int32, C.c_int32,
                                       _VP, C.c_double, _P(_VP)], C.c_int),
            "airg_dist_report": ([_VP, C.c_int64, _P(abi.LevelInfo), _P(C.c_int64)], C.c_int),
            "airg_dist_fused_nnz": ([_VP, C.c_int64, _P(C.c_int64), _P(C.c_int64)], C.c_int),
            "airg_dist_coarse_e_nnz": ([_VP, _P(C.c_int64)], C.c_int),
            "airg_dist_setup_times": ([_VP, _P(C.c_double), _P(C.c_double)], C.c_int),
            "airg_dist_create": ([_VP, _VP, C.c_int32, C.c_int32, _VP, C.c_double, _VP, _P(_VP)], C.c_int),
            "airg_dist_solve": ([_VP, _VP, _P(abi.SolveConfig), _VP, _VP, _P(abi.SolveStats), _VP,
                                 C.c_int64], C.c_int),
            "airg_dist_rank_bytes": ([_VP, C.c_int32, _P(C.c_int64)], C.c_int),
            "airg_dist_level_share": ([_VP, C.c_int64, _P(C.c_double), _P(C.c_double)], C.c_int),
            "airg_dist_halo_bytes": ([_VP, _P(abi.SolveConfig), _P(C.c_int64), _P(C.c_int64)], C.c_int),
            "airg_dist_level_info": ([_VP, C.c_int64, _P(C.c_int32), _P(C.c_double), _P(C.c_double),
                                      _P(C.c_int32), _P(C.c_int64), _VP], C.c_int),
            "airg_dist_transport": ([_VP, _P(C.c_int32)], C.c_int),
            "airg_p2p_push_plan_host": ([C.c_int32, _VP, C.c_int32, _VP, C.c_int64, C.c_int32, _VP, _VP,
                                         C.c_int64, _P(C.c_int64)], C.c_int),
            "airg_dist_destroy": ([_VP], C.c_int),
            "airg_mm_read": ([C.c_char_p, _P(_VP)], C.c_int),
            "airg_mm_dims": ([_VP, _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)], C.c_int),
            "airg_mm_copy": ([_VP, _VP, _VP, _VP], C.c_int),
            "airg_mm_free": ([_VP], C.c_int),
            "airg_mm_write": ([C.c_char_p, C.c_int64, C.c_int64, _VP, _VP, _VP], C.c_int),
            "airg_dist_cf_split": ([_VP, _VP, C.c_int32, C.c_int32, _VP, _VP, C.c_double, C.c_int64,
                                    C.c_uint64, C.c_int32, C.c_double, C.c_int64, _VP,
                                    _P(abi.CfReport)], C.c_int),
            "airg_dist_plan_host": ([C.c_int32, _VP, C.c_int32, _VP, C.c_int64, _VP, C.c_int64,
                                     _P(C.c_int64), _VP], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Every entry point include/airg_c.h declares (checked by the CPU tests)."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "airg_c.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(airg_[a-z0-9_]+)\s*\(", text)))


def _check(rc: int) -> None:
    if rc == 0:
        return
    buf = C.create_string_buffer(4096)
    lib().airg_last_error(buf, 4096)
    msg = buf.value.decode()
    if rc == -1:
        raise InvalidArgument(msg)
    if rc == -2:
        raise AirgRuntimeError(msg)
    raise CudaFailure(f"airg status {rc}: {msg}")


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


# ---------------------------------------------------------------------------
class Context:
    """One device + one stream (airg_ctx)."""

    def __init__(self, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise CudaFailure("no CUDA device: the AIRG engine runs on the GPU only")
        self.torch = torch
        self.device = device
        self.tdev = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=self.tdev)
        h = _VP()
        _check(lib().airg_ctx_create(device, C.byref(h)))
        self.h = h
        _check(lib().airg_ctx_set_stream(self.h, _VP(self.stream.cuda_stream)))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().airg_ctx_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def synchronize(self):
        _check(lib().airg_ctx_synchronize(self.h))

    def launches(self) -> int:
        v = C.c_uint64()
        _check(lib().airg_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    # device scratch on our stream
    def empty(self, n, dtype):
        with self.torch.cuda.stream(self.stream):
            return self.torch.empty(int(n), dtype=dtype, device=self.tdev)

    def to_device(self, a: np.ndarray):
        with self.torch.cuda.stream(self.stream):
            t = self.torch.from_numpy(np.ascontiguousarray(a)).to(self.tdev, non_blocking=False)
        return t

    def to_host(self, t) -> np.ndarray:
        self.stream.synchronize()
        return t.cpu().numpy()


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------------
@dataclass
class SparseMatrix:
    """Host CSR in the reference layout (sparse.hpp:33-94): int64 offsets
    and columns (strictly increasing per row), fp64 values."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @staticmethod
    def from_arrays(n, m, rp, ci, v) -> "SparseMatrix":
        return SparseMatrix(int(n), int(m), np.ascontiguousarray(rp, np.int64),
                            np.ascontiguousarray(ci, np.int64), np.ascontiguousarray(v, np.float64))

    @staticmethod
    def from_triplets(n, m, triplets) -> "SparseMatrix":
        """sparse.cpp:48-80 (duplicates summed in sorted order)."""
        rows = np.array([t[0] for t in triplets], np.int64)
        cols = np.array([t[1] for t in triplets], np.int64)
        vals = np.array([t[2] for t in triplets], np.float64)
        if len(rows) and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= m):
            raise InvalidArgument("SparseMatrix: triplet index out of range")
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        rp = np.zeros(n + 1, np.int64)
        oc, ov = [], []
        k = 0
        while k < len(rows):
            r, c, v = rows[k], cols[k], vals[k]
            k += 1
            while k < len(rows) and rows[k] == r and cols[k] == c:
                v += vals[k]
                k += 1
            oc.append(c)
            ov.append(v)
            rp[r + 1] += 1
        return SparseMatrix(n, m, np.cumsum(rp), np.array(oc, np.int64), np.array(ov, np.float64))

    @staticmethod
    def identity(n) -> "SparseMatrix":
        return SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))

    @staticmethod
    def diagonal(d) -> "SparseMatrix":
        n = len(d)
        return SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
                            np.asarray(d, np.float64).copy())

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.row_offsets[i], self.row_offsets[i + 1]
            d[i, self.col_indices[s:e]] = self.values[s:e]
        return d

    def __eq__(self, o) -> bool:  # exact comparison, sparse.hpp:87
        return (self.nrows == o.nrows and self.ncols == o.ncols
                and np.array_equal(self.row_offsets, o.row_offsets)
                and np.array_equal(self.col_indices, o.col_indices)
                and np.array_equal(self.values.view(np.uint64), o.values.view(np.uint64)))


class DeviceCSR:
    """An airg_csr handle (int32 indices, fp64 values, on the GPU)."""

    def __init__(self, ctx: Context, handle, owned: bool = True, keep=None):
        self.ctx, self.h, self.owned, self._keep = ctx, handle, owned, keep

    @staticmethod
    def upload(a: SparseMatrix, ctx: Context | None = None) -> "DeviceCSR":
        ctx = ctx or default_context()
        h = _VP()
        _check(lib().airg_csr_upload(ctx.h, a.nrows, a.ncols, a.row_offsets.ctypes.data,
                                     a.col_indices.ctypes.data, a.values.ctypes.data, C.byref(h)))
        return DeviceCSR(ctx, h)

    def __del__(self):
        if self.owned and getattr(self, "h", None):
            try:
                lib().airg_csr_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def dims(self):
        n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().airg_csr_info(self.h, C.byref(n), C.byref(m), C.byref(z)))
        return n.value, m.value, z.value

    def download(self) -> SparseMatrix:
        n, m, z = self.dims()
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(z, np.int64)
        v = np.zeros(z, np.float64)
        _check(lib().airg_csr_download(self.ctx.h, self.h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
        return SparseMatrix(n, m, rp, ci, v)


def _dev(a, ctx) -> DeviceCSR:
    return a if isinstance(a, DeviceCSR) else DeviceCSR.upload(a, ctx)


def _new(ctx, fn, *args) -> DeviceCSR:
    out = _VP()
    _check(fn(ctx.h, *args, C.byref(out)))
    return DeviceCSR(ctx, out)


def _new1(ctx, fn, d: DeviceCSR, *args) -> DeviceCSR:
    """Like _new with one matrix operand, kept alive across the call."""
    out = _VP()
    _check(fn(ctx.h, d.h, *args, C.byref(out)))
    return DeviceCSR(ctx, out)


# ---- L0 (sparse.hpp:97-110) -------------------------------------------------
def spmv(a, x, ctx: Context | None = None) -> np.ndarray:
    """y = A x (sparse.cpp:185-201); bit-identical to the reference."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    n, m, _ = d.dims()
    x = np.asarray(x, np.float64)
    if x.shape[0] != m:
        raise InvalidArgument("spmv: dimension mismatch")
    tx = ctx.to_device(x)
    ty = ctx.empty(n, ctx.torch.float64)
    _check(lib().airg_spmv(ctx.h, d.h, _ptr(tx), _ptr(ty)))
    return ctx.to_host(ty)


def spgemm(a, b, ctx: Context | None = None) -> SparseMatrix:
    """C = A B (sparse.cpp:203-242), cancellation zeros retained."""
    ctx = ctx or default_context()
    da, db = _dev(a, ctx), _dev(b, ctx)
    return _new(ctx, lib().airg_spgemm, da.h, db.h).download()


def drop_entries(a, tol: float, keep_diagonal: bool = True, ctx: Context | None = None) -> SparseMatrix:
    """sparse.cpp:244-268."""
    ctx = ctx or default_context()
    return _new1(ctx, lib().airg_drop, _dev(a, ctx), float(tol), int(keep_diagonal)).download()


def with_full_diagonal(a, ctx: Context | None = None) -> SparseMatrix:
    """SparseMatrix::with_full_diagonal (sparse.cpp:132-160)."""
    ctx = ctx or default_context()
    return _new1(ctx, lib().airg_with_full_diagonal, _dev(a, ctx)).download()


def extract_blocks(a, labels, ctx: Context | None = None):
    """sparse.cpp:292-340 -> (A_ff, A_fc, A_cf)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    tl = ctx.to_device(np.asarray(labels, np.uint8))
    o = [_VP(), _VP(), _VP()]
    _check(lib().airg_extract_blocks(ctx.h, d.h, _ptr(tl), C.byref(o[0]), C.byref(o[1]), C.byref(o[2])))
    return tuple(DeviceCSR(ctx, h).download() for h in o)


# ---- L1a (coarsening.hpp) ---------------------------------------------------------
def strength(a, alpha: float, ctx: Context | None = None) -> SparseMatrix:
    """coarsening.cpp:83-105: S as a pattern matrix (values 1.0)."""
    ctx = ctx or default_context()
    return _new1(ctx, lib().airg_strength, _dev(a, ctx), float(alpha)).download()


def pmisr(a, alpha: float, max_loops: int, seed: int, weight_mode: int = 0,
          ctx: Context | None = None):
    """strength -> pmisr (coarsening.cpp:107-167) -> (labels, weights)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    n = d.dims()[0]
    tl = ctx.empty(max(n, 1), ctx.torch.uint8)
    tw = ctx.empty(max(n, 1), ctx.torch.float64)
    _check(lib().airg_pmisr(ctx.h, d.h, float(alpha), int(max_loops), int(seed) & (2**64 - 1),
                            int(weight_mode), _ptr(tl), _ptr(tw)))
    return ctx.to_host(tl)[:n], ctx.to_host(tw)[:n]


def pmisr_with_weights(s_pattern: SparseMatrix, max_loops: int, weights,
                       ctx: Context | None = None) -> np.ndarray:
    """pmisr_with_weights (coarsening.cpp:107-160) on an explicit strength
    pattern (StrengthGraph::from_pattern) and explicit weights."""
    ctx = ctx or default_context()
    d = _dev(s_pattern, ctx)
    n = d.dims()[0]
    tw = ctx.to_device(np.asarray(weights, np.float64))
    tl = ctx.empty(max(n, 1), ctx.torch.uint8)
    _check(lib().airg_pmisr_with_weights(ctx.h, d.h, int(max_loops), _ptr(tw), _ptr(tl)))
    return ctx.to_host(tl)[:n]


def pmis(a, alpha=0.5, swap=False, seed=0, ctx: Context | None = None) -> np.ndarray:
    """pmis(strength(a, alpha), swap, seed) (coarsening.cpp:169-217): the
    classical PMIS / PMIS-swap baselines of the paper."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    n = d.dims()[0]
    tl = ctx.empty(max(n, 1), ctx.torch.uint8)
    _check(lib().airg_pmis(ctx.h, d.h, float(alpha), int(bool(swap)), int(seed) & (2**64 - 1), _ptr(tl)))
    return ctx.to_host(tl)[:n]


@dataclass
class CfReport:
    n_f_pre: int
    n_f: int
    n_c: int
    n_converted: int
    max_theta: float
    alpha_diag: float
    s_nnz: int


def cf_split(a, alpha=0.5, max_loops=3, seed=0, weight_mode=0, ddc_enabled=True,
             ddc_fraction=0.1, ddc_bins=1000, ctx: Context | None = None):
    """The fused split of air.cpp:466-494 -> (labels, pmisr_labels, report)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    n = d.dims()[0]
    tl = ctx.empty(max(n, 1), ctx.torch.uint8)
    tp = ctx.empty(max(n, 1), ctx.torch.uint8)
    rep = abi.CfReport()
    _check(lib().airg_cf_split(ctx.h, d.h, float(alpha), int(max_loops), int(seed) & (2**64 - 1),
                               int(weight_mode), int(ddc_enabled), float(ddc_fraction), int(ddc_bins),
                               _ptr(tl), _ptr(tp), C.byref(rep)))
    r = CfReport(rep.n_f_pre, rep.n_f, rep.n_c, rep.n_converted, rep.max_theta, rep.alpha_diag, rep.s_nnz)
    return ctx.to_host(tl)[:n], ctx.to_host(tp)[:n], r


def cf_split_device(d: DeviceCSR, alpha=0.5, max_loops=3, seed=0, weight_mode=0, ddc_enabled=True,
                    ddc_fraction=0.1, ddc_bins=1000, labels=None, ctx: Context | None = None):
    """cf_split on a device-resident matrix into a device label tensor."""
    ctx = ctx or d.ctx
    n = d.dims()[0]
    tl = labels if labels is not None else ctx.empty(max(n, 1), ctx.torch.uint8)
    rep = abi.CfReport()
    _check(lib().airg_cf_split(ctx.h, d.h, float(alpha), int(max_loops), int(seed) & (2**64 - 1),
                               int(weight_mode), int(ddc_enabled), float(ddc_fraction), int(ddc_bins),
                               _ptr(tl), None, C.byref(rep)))
    return tl, rep


def cf_split_batch_device(mats, seeds, alpha=0.5, max_loops=3, ddc_enabled=True, ddc_fraction=0.1,
                          ddc_bins=1000, labels=None, ctx: Context | None = None):
    """airg_cf_split_batch: cf_split (weight mode 0) of several device
    matrices with one synchronisation -> (device label tensors, reports)."""
    mats = list(mats)
    ctx = ctx or (mats[0].ctx if mats else default_context())
    k = len(mats)
    if labels is None:
        labels = [ctx.empty(max(m.dims()[0], 1), ctx.torch.uint8) for m in mats]
    hs = (_VP * max(k, 1))(*[m.h for m in mats])
    sd = np.asarray([int(x) & (2**64 - 1) for x in seeds], dtype=np.uint64)
    if len(sd) != k:
        raise ValueError("cf_split_batch: one seed per matrix")
    lp = (_VP * max(k, 1))(*[_ptr(t) for t in labels])
    reps = (abi.CfReport * max(k, 1))()
    _check(lib().airg_cf_split_batch(ctx.h, hs, k, sd.ctypes.data, float(alpha), int(max_loops),
                                     int(ddc_enabled), float(ddc_fraction), int(ddc_bins), lp, reps))
    return labels, [reps[i] for i in range(k)]


def spmv_device(d: DeviceCSR, tx, ty, ctx: Context | None = None) -> None:
    """y = A x on device tensors (no synchronisation)."""
    ctx = ctx or d.ctx
    _check(lib().airg_spmv(ctx.h, d.h, _ptr(tx), _ptr(ty)))


def ddc(a, labels, fraction=0.1, bins=1000, selection=0, direct_alpha_diag=0.0,
        ctx: Context | None = None):
    """coarsening.cpp:252-330 on the F block of A under `labels` (selection
    0 histogram, 2 direct) -> (new labels, report)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    tl = ctx.to_device(np.asarray(labels, np.uint8))
    rep = abi.CfReport()
    _check(lib().airg_ddc(ctx.h, d.h, _ptr(tl), float(fraction), int(bins), int(selection),
                          float(direct_alpha_diag), C.byref(rep)))
    return ctx.to_host(tl), rep


def dominance_report(a_ff, bins: int = 1000, ctx: Context | None = None):
    """coarsening.cpp:219-250 -> (theta, histogram (int64), max_theta)."""
    ctx = ctx or default_context()
    d = _dev(a_ff, ctx)
    n = d.dims()[0]
    tt = ctx.empty(max(n, 1), ctx.torch.float64)
    hist = np.zeros(max(int(bins), 1), np.int64)
    mx = C.c_double()
    _check(lib().airg_dominance_report(ctx.h, d.h, int(bins), _ptr(tt), hist.ctypes.data, C.byref(mx)))
    return ctx.to_host(tt)[:n], hist[: max(int(bins), 0)], mx.value


def build_label_map(labels, ctx: Context | None = None):
    """sparse.cpp:270-290 -> (fine_to_sub, f_to_fine, c_to_fine), int64."""
    ctx = ctx or default_context()
    lab = np.ascontiguousarray(labels, np.uint8)
    n = len(lab)
    tl = ctx.to_device(lab)
    nf = int(np.count_nonzero(lab == 0))
    f2s = np.zeros(max(n, 1), np.int64)
    f2f = np.zeros(max(nf, 1), np.int64)
    c2f = np.zeros(max(n - nf, 1), np.int64)
    out_nf = C.c_int64()
    _check(lib().airg_build_label_map(ctx.h, _ptr(tl), n, f2s.ctypes.data, f2f.ctypes.data, c2f.ctypes.data,
                                      C.byref(out_nf)))
    return f2s[:n], f2f[:nf], c2f[: n - nf]


def build_restriction(a_cf, aff_inv, drop_restrict: float, labels, ctx: Context | None = None) -> SparseMatrix:
    """air.cpp:154-189: R = [-drop(A_cf Aff_inv) | I] in fine columns."""
    ctx = ctx or default_context()
    dcf, dinv = _dev(a_cf, ctx), _dev(aff_inv, ctx)
    lab = np.ascontiguousarray(labels, np.uint8)
    tl = ctx.to_device(lab)
    out = _VP()
    _check(lib().airg_build_restriction(ctx.h, dcf.h, dinv.h, float(drop_restrict), _ptr(tl), len(lab),
                                        C.byref(out)))
    return DeviceCSR(ctx, out).download()


def build_prolongation(a, s_pattern, labels, ctx: Context | None = None) -> SparseMatrix:
    """air.cpp:191-238: one-point P from the strength pattern (strength(a, alpha))."""
    ctx = ctx or default_context()
    da, ds = _dev(a, ctx), _dev(s_pattern, ctx)
    tl = ctx.to_device(np.ascontiguousarray(labels, np.uint8))
    out = _VP()
    _check(lib().airg_build_prolongation(ctx.h, da.h, ds.h, _ptr(tl), C.byref(out)))
    return DeviceCSR(ctx, out).download()


def coarse_matrix(r, a, p, drop_coarse: float, ctx: Context | None = None) -> SparseMatrix:
    """air.cpp:268-271: drop_entries(R (A P), drop_coarse)."""
    ctx = ctx or default_context()
    dr, da, dp = _dev(r, ctx), _dev(a, ctx), _dev(p, ctx)
    out = _VP()
    _check(lib().airg_coarse_matrix(ctx.h, dr.h, da.h, dp.h, float(drop_coarse), C.byref(out)))
    return DeviceCSR(ctx, out).download()


# ---- L1b (gmres_poly.hpp) -----------------------------------------------------------
def apply_polynomial(a, coeffs, effective_order: int, b, ctx: Context | None = None) -> np.ndarray:
    """gmres_poly.cpp:173-195: q(A) b by Horner (effective_order matvecs)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    c = np.ascontiguousarray(coeffs, np.float64)
    n = d.dims()[0]
    tb = ctx.to_device(np.asarray(b, np.float64))
    ty = ctx.empty(max(n, 1), ctx.torch.float64)
    _check(lib().airg_apply_polynomial(ctx.h, d.h, c.ctypes.data, len(c), int(effective_order), _ptr(tb),
                                       _ptr(ty)))
    return ctx.to_host(ty)[:n]


def compute_coefficients(a, m: int, seed: int, ctx: Context | None = None):
    """gmres_poly.cpp:63-171 (double-double on the GPU) -> (coeffs, effective_order)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    out = np.zeros(max(int(m), 1))
    eff = C.c_int64()
    _check(lib().airg_poly_coefficients(ctx.h, d.h, int(m), int(seed) & (2**64 - 1),
                                        out.ctypes.data, C.byref(eff)))
    return out, eff.value


def assemble_fixed_sparsity(a, coeffs, effective_order: int, sparsity_order: int,
                            ctx: Context | None = None) -> SparseMatrix:
    """gmres_poly.cpp:197-280."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(coeffs, np.float64)
    return _new1(ctx, lib().airg_poly_assemble, _dev(a, ctx), c.ctypes.data, len(c),
                int(effective_order), int(sparsity_order)).download()


# ---- L2 / L3 (air.hpp, solve.hpp) ------------------------------------------------------
MATRICES = {"a": 0, "a_ff": 1, "a_fc": 2, "a_cf": 3, "ff_inv": 4, "r": 5, "p": 6, "afp": 7, "w": 8,
            "k": 9, "dsc": 10, "coarse_e": 9}


class Hierarchy:
    """A device-resident airgraph::Hierarchy (air.hpp:76-91)."""

    def __init__(self, ctx: Context, h, top_n: int, cfg: "abi.SetupConfig | None" = None):
        self.ctx, self.h, self.top_n = ctx, h, top_n
        cfg = cfg or abi.setup_config()
        self.coarse_poly_order = int(cfg.coarse_poly_order)  # GmresPolynomial::order of the coarse solver
        self.coarse_iterations = int(cfg.coarse_iterations)

    def __del__(self):
        self.close()

    def close(self):
        """Free the device hierarchy now (e.g. once a Dist holds its slabs)."""
        if getattr(self, "h", None):
            try:
                lib().airg_hier_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def info(self) -> abi.HierInfo:
        i = abi.HierInfo()
        _check(lib().airg_hier_info_get(self.h, C.byref(i)))
        return i

    @property
    def n_levels(self) -> int:
        return self.info().n_levels

    def level(self, l: int) -> abi.LevelInfo:
        i = abi.LevelInfo()
        _check(lib().airg_hier_level_info(self.h, int(l), C.byref(i)))
        return i

    def matrix(self, l: int, which) -> SparseMatrix:
        w = MATRICES[which] if isinstance(which, str) else int(which)
        out = _VP()
        _check(lib().airg_hier_matrix(self.h, int(l), w, C.byref(out)))
        return DeviceCSR(self.ctx, out, owned=False, keep=self).download()

    def fused_nnz(self, l: int) -> tuple[int, int]:
        """(nnz of A_F P, nnz of W) of the fast V-cycle's fused operators."""
        return (self.matrix_handle(l, 7).dims()[2], self.matrix_handle(l, 8).dims()[2])

    def fused_plan(self) -> dict:
        """Which levels run the fast V-cycle's one-pass ascent (K operator)
        and whether the coarse solve is composed (fused.cu)."""
        def has(l, w):
            try:
                self.matrix_handle(l, w)
                return True
            except InvalidArgument:
                return False
        return {"one_pass": [has(l, 9) for l in range(self.n_levels)],
                "coarse_composed": has(self.n_levels, 9)}

    def matrix_handle(self, l: int, which) -> DeviceCSR:
        """Borrowed device handle of a level matrix (no copy)."""
        w = MATRICES[which] if isinstance(which, str) else int(which)
        out = _VP()
        _check(lib().airg_hier_matrix(self.h, int(l), w, C.byref(out)))
        return DeviceCSR(self.ctx, out, owned=False, keep=self)

    def solve_host_ptr(self, hb: int, hx: int, **solve_kw) -> abi.SolveStats:
        """The host-buffer C-ABI solve on raw (pinned) host pointers."""
        cfg = abi.solve_config(**solve_kw)
        st = abi.SolveStats()
        _check(lib().airg_solve_host(self.ctx.h, self.h, C.byref(cfg), hb, hx, C.byref(st), None, 0))
        return st

    def labels(self, l: int) -> np.ndarray:
        n = self.level(l).n
        out = np.zeros(n, np.uint8)
        _check(lib().airg_hier_labels(self.ctx.h, self.h, int(l), out.ctypes.data))
        return out

    def f_smooth(self, level: int, b, x) -> np.ndarray:
        """f_smooth(level, b, x) (solve.cpp:63-87) -> the smoothed x."""
        tb = self.ctx.to_device(np.asarray(b, np.float64))
        tx = self.ctx.to_device(np.asarray(x, np.float64))
        _check(lib().airg_f_smooth(self.ctx.h, self.h, int(level), _ptr(tb), _ptr(tx)))
        return self.ctx.to_host(tx)

    def vcycle(self, b, **solve_kw) -> np.ndarray:
        """vcycle(h, b, x = 0) (solve.cpp:150-165)."""
        cfg = abi.solve_config(**solve_kw)
        tb = self.ctx.to_device(np.asarray(b, np.float64))
        tx = self.ctx.empty(self.top_n, self.ctx.torch.float64)
        _check(lib().airg_vcycle(self.ctx.h, self.h, C.byref(cfg), _ptr(tb), _ptr(tx)))
        return self.ctx.to_host(tx)

    def vcycle_device(self, tb, tx, **solve_kw) -> None:
        """One V-cycle x = M b with device-resident b / x (torch tensors)."""
        cfg = abi.solve_config(**solve_kw)
        _check(lib().airg_vcycle(self.ctx.h, self.h, C.byref(cfg), _ptr(tb), _ptr(tx)))

    def solve_device(self, tb, tx, history_cap: int = 0, **solve_kw):
        """Solve with device-resident b / x (torch tensors)."""
        cfg = abi.solve_config(**solve_kw)
        st = abi.SolveStats()
        hist = np.zeros(max(history_cap, 1))
        _check(lib().airg_solve(self.ctx.h, self.h, C.byref(cfg), _ptr(tb), _ptr(tx), C.byref(st),
                                hist.ctypes.data if history_cap else None, int(history_cap)))
        return st, hist[: min(history_cap, st.history_len)]


def _injection(injection: dict | None):
    """airg_injection from {"levels": [(coeffs, eff), ...], "coarse": (coeffs, eff)}
    (pointer, arrays to keep alive during the call)."""
    if injection is None:
        return None, []
    levels = injection["levels"]
    stride = 32
    lc = np.zeros(max(1, len(levels)) * stride)
    le = np.zeros(max(1, len(levels)), np.int64)
    for l, (co, eff) in enumerate(levels):
        lc[l * stride: l * stride + len(co)] = co
        le[l] = eff
    cc = np.zeros(32)
    cc[: len(injection["coarse"][0])] = injection["coarse"][0]
    inj = abi.Injection(len(levels), stride, lc.ctypes.data_as(_P(C.c_double)),
                        le.ctypes.data_as(_P(C.c_int64)), cc.ctypes.data_as(_P(C.c_double)),
                        int(injection["coarse"][1]))
    return C.byref(inj), [lc, le, cc, inj]


def setup(a, injection: dict | None = None, ctx: Context | None = None, nranks: int = 0, rank: int = -1,
          comm: "NcclComm | None" = None, **cfg_kw) -> Hierarchy:
    """airgraph::setup (air.cpp:285-410) on the GPU. `injection` (optional)
    = {"levels": [(coeffs, eff), ...], "coarse": (coeffs, eff)} takes the
    polynomial coefficients from the reference (coefficient-injection parity
    mode). nranks > 0: the setup's row work split over that
    many ranks (airg_dist_setup; rank = -1 emulates them all, rank >= 0 with
    a communicator is one rank of a torchrun job)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    cfg = abi.setup_config(**cfg_kw)
    inj_p, keep = _injection(injection)
    out = _VP()
    if nranks > 0:
        _check(lib().airg_dist_setup(ctx.h, d.h, C.byref(cfg), inj_p, int(nranks), int(rank),
                                     comm.h if comm else None, C.byref(out)))
    else:
        _check(lib().airg_setup(ctx.h, d.h, C.byref(cfg), inj_p, C.byref(out)))
    del keep
    return Hierarchy(ctx, out, d.dims()[0], cfg)


@dataclass
class SolveResult:
    x: np.ndarray
    stats: abi.SolveStats
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))


def richardson_solve(h: Hierarchy, b, history_cap: int = 1024, **solve_kw) -> SolveResult:
    """richardson_solve (solve.cpp:167-259) through the host-buffer C-ABI
    call (H2D of b, solve, D2H of x). outer=1 selects the outer GMRES."""
    cfg = abi.solve_config(**solve_kw)
    b = np.ascontiguousarray(b, np.float64)
    if b.shape[0] != h.top_n:
        raise InvalidArgument("richardson_solve: rhs length mismatch")
    x = np.zeros_like(b)
    st = abi.SolveStats()
    hist = np.zeros(history_cap)
    _check(lib().airg_solve_host(h.ctx.h, h.h, C.byref(cfg), b.ctypes.data, x.ctypes.data,
                                 C.byref(st), hist.ctypes.data, history_cap))
    return SolveResult(x, st, hist[: min(history_cap, st.history_len)])


def gmres_solve(h: Hierarchy, b, restart: int = 30, **solve_kw) -> SolveResult:
    """Right-preconditioned restarted GMRES with one AIRG V-cycle per
    iteration (BASELINE config 0's outer solver)."""
    return richardson_solve(h, b, outer=1, gmres_restart=restart, **solve_kw)


# ---- Matrix Market exchange (matrix_market.hpp:11-19) ----------------------------
def read_matrix_market(path) -> SparseMatrix:
    """airgraph::read_matrix_market: coordinate real general, duplicates summed
    exactly as the reference does (host code in the library; no GPU)."""
    h = _VP()
    _check(lib().airg_mm_read(os.fsencode(str(path)), C.byref(h)))
    try:
        n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().airg_mm_dims(h, C.byref(n), C.byref(m), C.byref(z)))
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(max(z.value, 1), np.int64)
        v = np.zeros(max(z.value, 1), np.float64)
        _check(lib().airg_mm_copy(h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
    finally:
        lib().airg_mm_free(h)
    return SparseMatrix(n.value, m.value, rp, ci[: z.value].copy(), v[: z.value].copy())


def write_matrix_market(a, path) -> None:
    """airgraph::write_matrix_market ("%.17g" values: exact round trip)."""
    if isinstance(a, DeviceCSR):
        a = a.download()
    rp = np.ascontiguousarray(a.row_offsets, np.int64)
    ci = np.ascontiguousarray(a.col_indices, np.int64)
    v = np.ascontiguousarray(a.values, np.float64)
    _check(lib().airg_mm_write(os.fsencode(str(path)), int(a.nrows), int(a.ncols), rp.ctypes.data,
                               ci.ctypes.data, v.ctypes.data))


# ---- multi-GPU: row-slab distributed solve ---------------------------
def plan_host(starts, rank: int, cols):
    """Host halo plan of one rank (no GPU): (sorted halo indices, recv counts per owner)."""
    s = np.ascontiguousarray(starts, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    P = len(s) - 1
    halo = np.zeros(max(1, len(c)), np.int64)
    nh = C.c_int64()
    rc = np.zeros(P, np.int64)
    _check(lib().airg_dist_plan_host(P, s.ctypes.data, int(rank), c.ctypes.data, len(c), halo.ctypes.data,
                                     len(halo), C.byref(nh), rc.ctypes.data))
    return halo[: nh.value].copy(), rc


def p2p_push_plan_host(starts, sender: int, recv_halo, receiver: int):
    """Host rule of the p2p push (no GPU): the entries of `receiver`'s sorted
    halo owned by `sender` -> (sender-local indices, positions in the
    receiver's [own | halo] buffer)."""
    s = np.ascontiguousarray(starts, np.int64)
    h = np.ascontiguousarray(recv_halo, np.int64)
    cap = max(1, len(h))
    si = np.zeros(cap, np.int32)
    pos = np.zeros(cap, np.int64)
    n = C.c_int64()
    _check(lib().airg_p2p_push_plan_host(len(s) - 1, s.ctypes.data, int(sender), h.ctypes.data, len(h),
                                         int(receiver), si.ctypes.data, pos.ctypes.data, cap, C.byref(n)))
    return si[: n.value].copy(), pos[: n.value].copy()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().airg_nccl_unique_id(buf))
    return buf.raw


class NcclComm:
    def __init__(self, nranks: int, rank: int, uid: bytes):
        buf = C.create_string_buffer(uid, 128)
        h = _VP()
        _check(lib().airg_nccl_comm_create(int(nranks), int(rank), buf, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().airg_nccl_comm_destroy(self.h)
            except Exception:
                pass
            self.h = None


def dist_cf_split_device(d: DeviceCSR, starts, rank: int = -1, comm: NcclComm | None = None, alpha=0.5,
                         max_loops=3, seed=0, ddc_enabled=True, ddc_fraction=0.1, ddc_bins=1000,
                         labels=None, ctx: Context | None = None):
    """Row-slab PMISR-DDC split (airg_dist_cf_split). rank = -1 emulates every
    slab in this process and returns global labels; rank >= 0 (with a
    communicator) returns this rank's slab. ``d`` is the global operator."""
    ctx = ctx or d.ctx
    s = np.ascontiguousarray(starts, np.int64)
    P = len(s) - 1
    n = d.dims()[0]
    cnt = n if rank < 0 else int(s[rank + 1] - s[rank])
    tl = labels if labels is not None else ctx.empty(max(cnt, 1), ctx.torch.uint8)
    rep = abi.CfReport()
    _check(lib().airg_dist_cf_split(ctx.h, d.h, P, int(rank), comm.h if comm else None, s.ctypes.data,
                                    float(alpha), int(max_loops), int(seed) & (2**64 - 1), int(ddc_enabled),
                                    float(ddc_fraction), int(ddc_bins), _ptr(tl), C.byref(rep)))
    r = CfReport(rep.n_f_pre, rep.n_f, rep.n_c, rep.n_converted, rep.max_theta, rep.alpha_diag, rep.s_nnz)
    return tl, r


def dist_cf_split(a, nranks: int, starts=None, alpha=0.5, max_loops=3, seed=0, ddc_enabled=True,
                  ddc_fraction=0.1, ddc_bins=1000, ctx: Context | None = None):
    """Emulated row-slab split of a host matrix -> (labels, report); equal
    slabs unless ``starts`` is given."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    n = d.dims()[0]
    if starts is None:
        starts = [n * r // nranks for r in range(nranks + 1)]
    tl, r = dist_cf_split_device(d, starts, -1, None, alpha, max_loops, seed, ddc_enabled, ddc_fraction,
                                 ddc_bins, ctx=ctx)
    return ctx.to_host(tl)[:n], r


class Dist:
    """A hierarchy partitioned into row slabs (airg_dist)."""

    def __init__(self, h: Hierarchy, nranks: int, rank: int = -1, comm: NcclComm | None = None,
                 threshold: float = 2.0, starts=None):
        self.h, self.ctx, self.P, self.rank = h, h.ctx, int(nranks), int(rank)
        st = None if starts is None else np.ascontiguousarray(starts, np.int64)
        self._starts = st
        out = _VP()
        _check(lib().airg_dist_create(self.ctx.h, h.h, self.P, self.rank, comm.h if comm else None,
                                      float(threshold), st.ctypes.data if st is not None else None,
                                      C.byref(out)))
        self.d = out
        self._comm = comm
        # level sizes kept here: the distribution owns its slabs, so the global
        # hierarchy may be closed once it exists (release_hierarchy)
        self.n_levels = h.n_levels
        self._levels = [(h.level(l).n, h.level(l).nnz) for l in range(self.n_levels)]
        hi = h.info()
        self._coarse = (hi.coarse_n, hi.coarse_nnz)

    @classmethod
    def setup_owned(cls, a, nranks: int, rank: int = -1, comm: NcclComm | None = None, threshold: float = 2.0,
                    starts=None, injection: dict | None = None, ctx: Context | None = None, **cfg_kw) -> "Dist":
        """Owned-row distributed setup (airg_dist_setup_owned): every rank
        builds and keeps only its rows of every level. rank = -1 emulates all
        ranks from the whole operator `a`; rank >= 0 (one process per GPU,
        with `comm`) takes this rank's rows starts[rank].. with global
        columns. starts defaults to balanced slabs of the global size."""
        ctx = ctx or default_context()
        d = _dev(a, ctx)
        n_glob = d.dims()[1]
        P = int(nranks)
        if starts is None:
            base, extra = divmod(n_glob, P)
            starts = np.concatenate([[0], np.cumsum([base + (1 if r < extra else 0) for r in range(P)])])
        st = np.ascontiguousarray(starts, np.int64)
        cfg = abi.setup_config(**cfg_kw)
        inj_p, keep = _injection(injection)
        out = _VP()
        _check(lib().airg_dist_setup_owned(ctx.h, d.h, st.ctypes.data, C.byref(cfg), inj_p, P, int(rank),
                                           comm.h if comm else None, float(threshold), C.byref(out)))
        del keep
        self = cls.__new__(cls)
        self.h, self.ctx, self.P, self.rank = None, ctx, P, int(rank)
        self._starts = st
        self.d = out
        self._comm = comm
        nl = C.c_int64()
        _check(lib().airg_dist_report(self.d, 0, None, C.byref(nl)))
        self.n_levels = nl.value
        reps = [self.report(l) for l in range(self.n_levels + 1)]
        self._levels = [(r.n, r.nnz) for r in reps[:-1]]
        self._coarse = (reps[-1].n, reps[-1].nnz)
        return self

    def report(self, l: int) -> abi.LevelInfo:
        """Setup report of level l of an owned distribution (l = n_levels: the
        coarse grid; airg_dist_report)."""
        info = abi.LevelInfo()
        _check(lib().airg_dist_report(self.d, int(l), C.byref(info), None))
        return info

    def setup_times(self) -> tuple[float, float]:
        """(wall ms of the owned setup, device ms of its CF splits) on this process."""
        a, b = C.c_double(), C.c_double()
        _check(lib().airg_dist_setup_times(self.d, C.byref(a), C.byref(b)))
        return a.value, b.value

    def release_hierarchy(self):
        """Drop this distribution's reference to the global hierarchy: only
        the per-rank slabs stay resident (call h.close() to free it now)."""
        self.h = None

    def fused_nnz(self, l: int) -> tuple[int, int]:
        """Global entries of the fast V-cycle's (A_F P, W_k) slabs of level l."""
        a, w = C.c_int64(), C.c_int64()
        _check(lib().airg_dist_fused_nnz(self.d, int(l), C.byref(a), C.byref(w)))
        return a.value, w.value

    def coarse_e_nnz(self) -> int:
        """Entries of the composed coarse solve held by this process (-1: not used)."""
        v = C.c_int64()
        _check(lib().airg_dist_coarse_e_nnz(self.d, C.byref(v)))
        return v.value

    def rank_bytes(self, rank: int | None = None) -> int:
        """Device bytes of one rank's slabs (airg_dist_rank_bytes)."""
        b = C.c_int64()
        _check(lib().airg_dist_rank_bytes(self.d, int(self.rank if rank is None else rank), C.byref(b)))
        return b.value

    def __del__(self):
        if getattr(self, "d", None):
            try:
                lib().airg_dist_destroy(self.d)
            except Exception:
                pass
            self.d = None

    @property
    def transport(self) -> str:
        """Halo transport of the solve: "gather" (emulation), "nccl" or "p2p"."""
        t = C.c_int32()
        _check(lib().airg_dist_transport(self.d, C.byref(t)))
        return ("gather", "nccl", "p2p")[t.value]

    def level_info(self, l: int) -> dict:
        a, t = C.c_int32(), C.c_int32()
        rb, ra = C.c_double(), C.c_double()
        halo = C.c_int64()
        starts = np.zeros(self.P + 1, np.int64)
        _check(lib().airg_dist_level_info(self.d, int(l), C.byref(a), C.byref(rb), C.byref(ra), C.byref(t),
                                          C.byref(halo), starts.ctypes.data))
        out = dict(active=a.value, ratio_before=rb.value, ratio_after=ra.value, triggered=bool(t.value),
                   halo=halo.value, starts=starts)
        if l < self.n_levels:
            sb, sa = C.c_double(), C.c_double()
            _check(lib().airg_dist_level_share(self.d, int(l), C.byref(sb), C.byref(sa)))
            out.update(share_before=sb.value, share_after=sa.value)
        return out

    def halo_bytes(self, **solve_kw) -> tuple[int, int]:
        """(bytes per V-cycle, bytes per level-0 SpMV) of halo data this
        process receives (NVLink traffic of the solve)."""
        cfg = abi.solve_config(**solve_kw)
        v, s = C.c_int64(), C.c_int64()
        _check(lib().airg_dist_halo_bytes(self.d, C.byref(cfg), C.byref(v), C.byref(s)))
        return v.value, s.value

    def solve_device(self, tb, tx, history_cap: int = 0, **solve_kw):
        cfg = abi.solve_config(**solve_kw)
        st = abi.SolveStats()
        hist = np.zeros(max(history_cap, 1))
        _check(lib().airg_dist_solve(self.ctx.h, self.d, C.byref(cfg), _ptr(tb), _ptr(tx), C.byref(st),
                                     hist.ctypes.data if history_cap else None, int(history_cap)))
        return st, hist[: min(history_cap, st.history_len)]

    def solve(self, b, **solve_kw):
        """Emulated (rank = -1): global host b -> global host x."""
        tb = self.ctx.to_device(np.asarray(b, np.float64))
        tx = self.ctx.empty(len(b), self.ctx.torch.float64)
        st, hist = self.solve_device(tb, tx, history_cap=1024, **solve_kw)
        return SolveResult(self.ctx.to_host(tx), st, hist)
