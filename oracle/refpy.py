"""ctypes bindings for the oracles -- TEST INFRASTRUCTURE ONLY.

Two CPU checkers with one Python surface:
  * RefLib  -- oracle/_ref/libairgraph_ref.so: the UNMODIFIED reference
    sources compiled from /root/reference (oracle/Makefile `ref`), driven
    through oracle/ref_capi.cpp.
  * PortLib -- oracle/liboracle.so: the C restatement oracle/airg_oracle.c
    (oracle/Makefile `port`), which exists everywhere (the GPU box has no
    /root/reference).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

import sys  # noqa: E402

if REPO not in sys.path:
    sys.path.insert(0, REPO)
from paper_2408_08262_b200 import abi  # noqa: E402  (shared ctypes structs)

i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class OracleValueError(ValueError):
    pass


def build_port() -> str:
    path = os.path.join(HERE, "liboracle.so")
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return path


def build_ref() -> str | None:
    if not os.path.isdir("/root/reference/proj/src"):
        return None
    subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)
    return os.path.join(HERE, "_ref", "libairgraph_ref.so")


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        for name, args in [
            ("last_error", [C.c_char_p, C.c_size_t]),
            ("mat_new", [C.c_int64, C.c_int64, i64p, i64p, f64p, C.POINTER(C.c_void_p)]),
            ("mat_dims", [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            ("mat_copy", [C.c_void_p, i64p, i64p, f64p]),
            ("mat_free", [C.c_void_p]),
            ("spmv", [C.c_void_p, f64p, f64p]),
            ("spgemm", [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
            ("drop", [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
            ("with_full_diagonal", [C.c_void_p, C.POINTER(C.c_void_p)]),
            ("extract_blocks", [C.c_void_p, u8p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
            ("strength", [C.c_void_p, C.c_double, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
            ("pmisr", [C.c_void_p, C.c_double, C.c_int64, C.c_uint64, C.c_int32, u8p, C.c_void_p]),
            ("pmisr_with_weights", [C.c_void_p, C.c_int64, f64p, u8p]),
            ("cf_split", [C.c_void_p, C.c_double, C.c_int64, C.c_uint64, C.c_int32, C.c_int32,
                          C.c_double, C.c_int64, u8p, C.c_void_p, C.POINTER(abi.CfReport)]),
            ("ddc", [C.c_void_p, u8p, C.c_double, C.c_int64, C.c_int32, C.c_double, C.POINTER(abi.CfReport)]),
            ("poly_coefficients", [C.c_void_p, C.c_int64, C.c_uint64, f64p, C.POINTER(C.c_int64)]),
            ("poly_assemble", [C.c_void_p, f64p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
            ("setup", [C.c_void_p, C.POINTER(abi.SetupConfig), C.POINTER(C.c_void_p)]),
            ("hier_free", [C.c_void_p]),
            ("hier_info", [C.c_void_p, C.POINTER(abi.HierInfo)]),
            ("level_info", [C.c_void_p, C.c_int64, C.POINTER(abi.LevelInfo)]),
            ("hier_matrix", [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]),
            ("hier_labels", [C.c_void_p, C.c_int64, u8p]),
            ("vcycle", [C.c_void_p, C.POINTER(abi.SolveConfig), f64p, f64p]),
            ("solve", [C.c_void_p, C.POINTER(abi.SolveConfig), f64p, f64p, C.POINTER(abi.SolveStats), f64p, C.c_int64]),
            ("dominance_report", [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
            ("build_label_map", [u8p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
            ("build_restriction", [C.c_void_p, C.c_void_p, C.c_double, u8p, C.c_int64, C.POINTER(C.c_void_p)]),
            ("build_prolongation", [C.c_void_p, C.c_void_p, u8p, C.POINTER(C.c_void_p)]),
            ("coarse_matrix", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(C.c_void_p)]),
            ("apply_polynomial", [C.c_void_p, f64p, C.c_int64, C.c_int64, f64p, f64p]),
            ("f_smooth", [C.c_void_p, C.c_int64, f64p, f64p]),
        ]:
            fn = getattr(L, p + name, None)
            if fn is None:
                continue
            fn.argtypes = args
            fn.restype = C.c_int
        self.has_desk = hasattr(L, p + "desk_problem")
        if self.has_desk:
            fn = getattr(L, p + "desk_problem")
            fn.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.POINTER(C.c_void_p), f64p, C.c_int64, C.POINTER(C.c_int64)]
            fn.restype = C.c_int

    # -- helpers -----------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _chk(self, rc):
        if rc == 0:
            return
        buf = C.create_string_buffer(4096)
        self._fn("last_error")(buf, 4096)
        msg = buf.value.decode()
        if rc == -1:
            raise OracleValueError(msg)
        raise OracleError(msg)

    def call(self, name, *args):
        self._chk(self._fn(name)(*args))

    # -- matrices -----------------------------------------------------------
    def mat(self, n, m, rp, ci, v) -> "Mat":
        h = C.c_void_p()
        self.call("mat_new", n, m, np.ascontiguousarray(rp, np.int64),
                  np.ascontiguousarray(ci, np.int64), np.ascontiguousarray(v, np.float64), C.byref(h))
        return Mat(self, h, owned=True)

    def mat_from_problem(self, p) -> "Mat":
        return self.mat(p.n, p.n, p.row_offsets, p.cols, p.vals)


class Mat:
    """A handle to a SparseMatrix living in one of the oracle libraries."""

    def __init__(self, lib: _Lib, h, owned: bool):
        self.lib, self.h, self.owned = lib, h, owned

    def __del__(self):
        if self.owned and self.h:
            try:
                self.lib._fn("mat_free")(self.h)
            except Exception:
                pass

    def dims(self):
        n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib._fn("mat_dims")(self.h, C.byref(n), C.byref(m), C.byref(z))
        return n.value, m.value, z.value

    def arrays(self):
        n, m, z = self.dims()
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(z, np.int64)
        v = np.zeros(z, np.float64)
        self.lib._fn("mat_copy")(self.h, rp, ci, v)
        return rp, ci, v

    def to_dict(self):
        n, m, z = self.dims()
        rp, ci, v = self.arrays()
        return dict(n=n, m=m, rp=rp, ci=ci, v=v)


class RefLib(_Lib):
    prefix = "ref_"

    # matrix_market.hpp:11-19 (reference build only). The reference's reader
    # crashes inside a process that has imported numpy (a C++ runtime clash
    # around std::filesystem / iostreams in this image), so both calls run in
    # a numpy-free child interpreter that exchanges raw arrays through files.
    _MM_CHILD = r"""
import ctypes as C, struct, sys
L = C.CDLL(sys.argv[1])
op, path, blob = sys.argv[2], sys.argv[3], sys.argv[4]
buf = C.create_string_buffer(4096)
def chk(rc):
    if rc:
        L.ref_last_error(buf, 4096)
        sys.stderr.write(buf.value.decode()); sys.exit(3)
h = C.c_void_p()
if op == "read":
    L.ref_mm_read.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    chk(L.ref_mm_read(path.encode(), C.byref(h)))
    n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
    L.ref_mat_dims(h, C.byref(n), C.byref(m), C.byref(z))
    rp = (C.c_int64 * (n.value + 1))(); ci = (C.c_int64 * max(z.value, 1))(); v = (C.c_double * max(z.value, 1))()
    L.ref_mat_copy(h, rp, ci, v)
    with open(blob, "wb") as f:
        f.write(struct.pack("<3q", n.value, m.value, z.value))
        f.write(bytes(rp)); f.write(bytes(ci)[: 8 * z.value]); f.write(bytes(v)[: 8 * z.value])
else:
    with open(blob, "rb") as f:
        n, m, z = struct.unpack("<3q", f.read(24))
        rp = (C.c_int64 * (n + 1)).from_buffer_copy(f.read(8 * (n + 1)))
        ci = (C.c_int64 * max(z, 1)).from_buffer_copy(f.read(8 * z).ljust(8, b"\0"))
        v = (C.c_double * max(z, 1)).from_buffer_copy(f.read(8 * z).ljust(8, b"\0"))
    L.ref_mat_new.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
    chk(L.ref_mat_new(n, m, rp, ci, v, C.byref(h)))
    L.ref_mm_write.argtypes = [C.c_void_p, C.c_char_p]
    chk(L.ref_mm_write(h, path.encode()))
"""

    def _mm_child(self, op, path, blob):
        import sys as _sys
        r = subprocess.run([_sys.executable, "-c", self._MM_CHILD, self.path, op, str(path), str(blob)],
                           capture_output=True, text=True)
        if r.returncode == 3:
            raise OracleError(r.stderr)
        if r.returncode:
            raise RuntimeError(f"reference matrix-market child failed: {r.stderr[-500:]}")

    def mm_read(self, path: str):
        """-> (nrows, ncols, row_offsets, col_indices, values)"""
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            blob = os.path.join(d, "m.bin")
            self._mm_child("read", path, blob)
            raw = open(blob, "rb").read()
        n, m, z = np.frombuffer(raw[:24], np.int64)
        o = 24
        rp = np.frombuffer(raw[o:o + 8 * (n + 1)], np.int64).copy()
        o += 8 * (n + 1)
        ci = np.frombuffer(raw[o:o + 8 * z], np.int64).copy()
        o += 8 * z
        v = np.frombuffer(raw[o:o + 8 * z], np.float64).copy()
        return int(n), int(m), rp, ci, v

    def mm_write(self, a: Mat, path: str) -> None:
        import tempfile
        n, m, z = a.dims()
        rp, ci, v = a.arrays()
        with tempfile.TemporaryDirectory() as d:
            blob = os.path.join(d, "m.bin")
            with open(blob, "wb") as f:
                f.write(np.array([n, m, z], np.int64).tobytes())
                f.write(rp.tobytes())
                f.write(ci.tobytes())
                f.write(v.tobytes())
            self._mm_child("write", path, blob)


class PortLib(_Lib):
    prefix = "orc_"


_ref = None
_port = None


def ref() -> RefLib | None:
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libairgraph_ref.so")
        if not os.path.exists(path):
            path = build_ref()
        if path is None or not os.path.exists(path):
            return None
        _ref = RefLib(path)
    return _ref


def port() -> PortLib:
    global _port
    if _port is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build_port()
        _port = PortLib(path)
    return _port


# ---- high-level operations shared by both libraries -----------------------
def new_out():
    return C.c_void_p()


def spmv(lib, A: Mat, x):
    n, m, _ = A.dims()
    x = np.ascontiguousarray(x, np.float64)
    if x.shape[0] != m:  # sparse.cpp:187-188
        raise OracleValueError("spmv: dimension mismatch")
    y = np.zeros(n)
    lib.call("spmv", A.h, x, y)
    return y


def binop(lib, name, *args):
    out = C.c_void_p()
    lib.call(name, *args, C.byref(out))
    return Mat(lib, out, owned=True)


def cf_split(lib, A: Mat, cfg: dict, seed: int):
    cfg = {**abi.SETUP_DEFAULTS, **cfg}
    n = A.dims()[0]
    lab = np.zeros(n, np.uint8)
    pre = np.zeros(n, np.uint8)
    rep = abi.CfReport()
    lib.call("cf_split", A.h, cfg["strength_alpha"], cfg["max_loops"], seed, cfg.get("weight_mode", 0),
             cfg.get("ddc_enabled", 1), cfg["ddc_fraction"], cfg["ddc_bins"], lab,
             pre.ctypes.data_as(C.c_void_p), C.byref(rep))
    return lab, pre, rep


class Hier:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if self.h:
            try:
                self.lib._fn("hier_free")(self.h)
            except Exception:
                pass

    def info(self):
        i = abi.HierInfo()
        self.lib.call("hier_info", self.h, C.byref(i))
        return i

    def level(self, l):
        i = abi.LevelInfo()
        self.lib.call("level_info", self.h, l, C.byref(i))
        return i

    def matrix(self, l, which) -> Mat:
        out = C.c_void_p()
        self.lib.call("hier_matrix", self.h, l, which, C.byref(out))
        m = Mat(self.lib, out, owned=False)
        m._keep = self
        return m

    def report(self) -> str:
        """reports.cpp hierarchy_report(h).dump() (reference build only)."""
        f = self.lib.lib.ref_hier_report
        f.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
        n = C.c_int64()
        self.lib._chk(f(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.lib._chk(f(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def partition_report(self, ranks: int, threshold: float) -> str:
        """reports.cpp partition_report(replay_triggers(h, ranks, threshold))
        (reference build only)."""
        f = self.lib.lib.ref_partition_report
        f.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
        n = C.c_int64()
        self.lib._chk(f(self.h, int(ranks), float(threshold), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.lib._chk(f(self.h, int(ranks), float(threshold), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def csv_row(self, st, alpha, cf_name, seed) -> str:
        f = self.lib.lib.ref_csv_row
        f.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_int32, C.c_double, C.c_double, C.c_char_p,
                      C.c_uint64, C.c_char_p, C.c_int64]
        buf = C.create_string_buffer(1024)
        self.lib._chk(f(self.h, int(st.iterations), float(st.work_units), int(bool(st.converged)),
                        float(st.final_relative_residual), float(alpha), cf_name.encode(), int(seed), buf, 1024))
        return buf.value.decode()

    def labels(self, l):
        n = self.level(l).n
        out = np.zeros(n, np.uint8)
        self.lib.call("hier_labels", self.h, l, out)
        return out

    def f_smooth(self, level, b, x):
        """One F-smooth on `level` (solve.cpp:63-87) -> the smoothed x."""
        xx = np.ascontiguousarray(x, np.float64).copy()
        self.lib.call("f_smooth", self.h, int(level), np.ascontiguousarray(b, np.float64), xx)
        return xx

    def vcycle(self, b, scfg=None):
        scfg = scfg or abi.solve_config()
        x = np.zeros_like(b)
        self.lib.call("vcycle", self.h, C.byref(scfg), np.ascontiguousarray(b, np.float64), x)
        return x

    def solve(self, b, scfg=None, cap=1000):
        scfg = scfg or abi.solve_config()
        x = np.zeros_like(b)
        st = abi.SolveStats()
        hist = np.zeros(cap)
        self.lib.call("solve", self.h, C.byref(scfg), np.ascontiguousarray(b, np.float64), x,
                      C.byref(st), hist, cap)
        return x, st, hist[: min(cap, st.history_len)]


def setup(lib, A: Mat, **params) -> Hier:
    cfg = abi.setup_config(**params)
    out = C.c_void_p()
    lib.call("setup", A.h, C.byref(cfg), C.byref(out))
    return Hier(lib, out)


# ---- single reference operations (both libraries, same shapes) -------------
def dominance_report(lib, A: Mat, bins: int):
    n = A.dims()[0]
    theta = np.zeros(max(n, 1))
    hist = np.zeros(bins, np.int64)
    mx = C.c_double()
    lib.call("dominance_report", A.h, int(bins), theta.ctypes.data, hist.ctypes.data, C.byref(mx))
    return theta[:n], hist, mx.value


def build_label_map(lib, labels):
    lab = np.ascontiguousarray(labels, np.uint8)
    n = len(lab)
    nf = int(np.count_nonzero(lab == 0))
    f2s = np.zeros(max(n, 1), np.int64)
    f2f = np.zeros(max(nf, 1), np.int64)
    c2f = np.zeros(max(n - nf, 1), np.int64)
    out_nf = C.c_int64()
    lib.call("build_label_map", lab, n, f2s.ctypes.data, f2f.ctypes.data, c2f.ctypes.data, C.byref(out_nf))
    return f2s[:n], f2f[:nf], c2f[: n - nf]


def apply_polynomial(lib, A: Mat, coeffs, eff: int, b):
    c = np.ascontiguousarray(coeffs, np.float64)
    bb = np.ascontiguousarray(b, np.float64)
    y = np.zeros(max(A.dims()[0], 1))
    lib.call("apply_polynomial", A.h, c, len(c), int(eff), bb, y)
    return y[: A.dims()[0]]
