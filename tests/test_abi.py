"""CPU checks of the drop-in boundary: the sm_100a library loads, exports
every entry point include/airg_c.h declares, the ctypes mirrors match the C
struct layout, and the product fails loudly without a GPU (no CPU fallback).
"""
import ctypes as C
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2408_08262_b200 import abi, airg

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    L = airg.lib()
    syms = airg.exported_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", airg.LIB_PATH],
                         capture_output=True, text=True)
    assert out.returncode == 0 and "sm_100a" in out.stdout


def test_struct_layouts_match_header():
    structs = {"airg_setup_config": abi.SetupConfig, "airg_solve_config": abi.SolveConfig,
               "airg_solve_stats": abi.SolveStats, "airg_level_info": abi.LevelInfo,
               "airg_hier_info": abi.HierInfo, "airg_cf_report": abi.CfReport,
               "airg_injection": abi.Injection}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "airg_c.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        open(src, "w").write("\n".join(lines))
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(line.split() for line in out if line)
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"


def test_defaults_match_reference():
    cfg = abi.SetupConfig()
    airg.lib().airg_setup_config_default(C.byref(cfg))
    for k, v in abi.SETUP_DEFAULTS.items():  # air.hpp:16-43
        assert getattr(cfg, k) == pytest.approx(v), k
    s = abi.SolveConfig()
    airg.lib().airg_solve_config_default(C.byref(s))
    for k, v in abi.SOLVE_DEFAULTS.items():  # solve.hpp:11-19
        assert getattr(s, k) == pytest.approx(v), k


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(airg.CudaFailure):
        airg.spmv(airg.SparseMatrix.identity(3), np.ones(3))
    h = C.c_void_p()
    rc = airg.lib().airg_ctx_create(0, C.byref(h))
    assert rc != 0


def test_error_text_is_thread_local_and_readable():
    cfg = abi.SetupConfig()
    rc = airg.lib().airg_setup(None, None, C.byref(cfg), None, C.byref(C.c_void_p()))
    assert rc == -1
    buf = C.create_string_buffer(256)
    airg.lib().airg_last_error(buf, 256)
    assert b"null" in buf.value
