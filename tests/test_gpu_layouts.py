"""Every row-kernel decomposition gives the same bits (tiled.cuh): thread per
row, G-lane groups (G = 2..32), warp tiles, SELL-32/G, shared-memory staged
slices and long-row lane groups, selected by
environment variables that are read once per process -- hence one
subprocess per layout. Each prints the SHA-256 of the solution's bytes of a
reduced C2 solve and of a level-0 SpMV."""
import os
import subprocess
import sys

import pytest

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

LAYOUTS = {
    "thread": {"AIRG_ROWS": "thread", "AIRG_VEC": "0", "AIRG_TAIL_N": "0"},
    "vec4": {"AIRG_VEC": "4"},
    "vec8": {"AIRG_VEC": "8"},
    "short4": {"AIRG_VEC": "4"},
    "group_auto": {"AIRG_ROWS": "group"},
    "g2": {"AIRG_GROUP": "2"},
    "g4": {"AIRG_GROUP": "4"},
    "g8": {"AIRG_GROUP": "8"},
    "g16": {"AIRG_GROUP": "16"},
    "g32": {"AIRG_GROUP": "32"},
    "tiles": {"AIRG_ROWS": "tiles"},
    "sell": {"AIRG_LAYOUT": "sell"},
    "nopdl": {"AIRG_PDL": "0"},
    "early_fres1": {"AIRG_EARLY": "1"},
    "split_fres1": {"AIRG_SPLIT": "1"},
    "sorted_rows": {"AIRG_SORT": "1"},
    "c16": {"AIRG_C16": "1"},
    "tail_off": {"AIRG_TAIL_N": "0"},
    "tail_cluster_all": {"AIRG_TAIL": "cluster", "AIRG_TAIL_N": "100000000"},
    "tail_cluster_small": {"AIRG_TAIL": "cluster", "AIRG_TAIL_N": "2000"},
    "tail_grid_all": {"AIRG_TAIL": "grid", "AIRG_TAIL_N": "100000000"},
    "staged": {"AIRG_STAGE": "1"},
    "staged_small_cap": {"AIRG_STAGE": "1", "AIRG_STAGE_CAP": "64"},
    "wg4_all": {"AIRG_WG": "4", "AIRG_WG_ROWS": "1"},
    "wg8": {"AIRG_WG": "8"},
    "wg16_all": {"AIRG_WG": "16", "AIRG_WG_ROWS": "1"},
    "w32": {"AIRG_W32": "1"},
    "w32_all": {"AIRG_W32": "1", "AIRG_W32_ROWS": "1"},
}


def _run(env_extra):
    env = dict(os.environ)
    for k in ("AIRG_ROWS", "AIRG_GROUP", "AIRG_LAYOUT", "AIRG_PDL", "AIRG_VEC", "AIRG_TAIL_N", "AIRG_TAIL",
              "AIRG_DEVLOOP", "AIRG_EARLY", "AIRG_SPLIT", "AIRG_SORT",
              "AIRG_C16", "AIRG_STAGE", "AIRG_STAGE_CAP", "AIRG_WG", "AIRG_WG_ROWS", "AIRG_W32", "AIRG_W32_ROWS"):
        env.pop(k, None)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.strip().split("\n")[-1]


def test_all_layouts_bit_identical():
    base = _run(LAYOUTS["thread"])
    for name, env in LAYOUTS.items():
        if name != "thread":
            assert _run(env) == base, f"layout {name} differs from thread-per-row"


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
    "fused_g4": {"AIRG_CF_GROUP": "4"},
    "fused_g8": {"AIRG_CF_GROUP": "8"},
    "fused_g16": {"AIRG_CF_GROUP": "16"},
    "fused_default": {},
    "fused_no_small": {"AIRG_CF_SMALL": "0"},
    "fused_all_small": {"AIRG_CF_SMALL": "1000000000"},
    "fused_all_small_scalar": {"AIRG_CF_SMALL": "1000000000", "AIRG_CF_VEC": "100000"},
}


def test_cf_split_variants_bit_identical():
    """The fused split's variants (scalar, 16-byte loads, G lanes per row,
    the one-launch small-level split on no / every level) and the
    step-by-step split give the same hierarchy labels and
    DDC reports on every level (C2/C3/C4, reduced)."""
    def run(extra):
        env = dict(os.environ)
        for k in ("AIRG_CF", "AIRG_CF_VEC", "AIRG_CF_GROUP", "AIRG_CF_SMALL"):
            env.pop(k, None)
        env.update(extra)
        out = subprocess.run([sys.executable, "-c", CF_SCRIPT], env=env, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        return out.stdout.strip().split("\n")[-1]
    base = run(CF_VARIANTS["legacy"])
    for name, env in CF_VARIANTS.items():
        if name != "legacy":
            assert run(env) == base, f"CF variant {name} differs from the step-by-step split"
