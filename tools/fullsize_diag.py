"""Native-mode setup vs the reference's full-size fixtures: per level, where
the GPU's double-double coefficient fit leads to a different hierarchy.
  python tools/fullsize_diag.py [configs...]   (GPU)"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

FULL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "full")


def dg(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
    g = np.load(os.path.join(FULL, f"c{cfg}.npz"))
    p = problems.make(cfg)
    prm = eval(str(g["params"][0]))
    h = airg.setup(airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals), **prm)
    print(f"C{cfg}: levels gpu {h.n_levels} ref {int(g['n_levels'])}  coarse gpu {h.info().coarse_n} "
          f"ref {int(g['coarse_n'])}")
    for l in range(max(h.n_levels, int(g["n_levels"]))):
        if l >= h.n_levels or l >= int(g["n_levels"]):
            print(f"  {l:2d} only in {'ref' if l >= h.n_levels else 'gpu'}")
            continue
        L = h.level(l)
        same = dg(h.labels(l)) == str(g["level_labels_digest"][l])
        c1 = np.array(L.coefficients[: prm["poly_order"] + 1])
        c2 = g["level_coeffs"][l]
        print(f"  {l:2d} n {L.n:8d}/{g['level_n'][l]:8d} nnz {L.nnz:9d}/{g['level_nnz'][l]:9d} "
              f"nf {L.n_f:8d}/{g['level_nf'][l]:8d} eff {L.effective_order}/{g['level_eff'][l]} "
              f"att {L.poly_attempts}/{g['level_attempts'][l]} growth {L.smoother_growth:.9f}/"
              f"{g['level_growth'][l]:.9f} coef {np.abs(c1 - c2).max() / max(1, np.abs(c2).max()):.1e} "
              f"labels {'same' if same else 'DIFF'}")
    sys.stdout.flush()
