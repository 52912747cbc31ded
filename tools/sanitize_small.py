"""Small end-to-end run for compute-sanitizer (memcheck / racecheck /
synccheck): setup, the fused CF split, Richardson and GMRES solves in exact
and fast mode (fused level operators, device-resident GMRES), distributed
emulation (Richardson and GMRES). AIRG_GM_FLAT=1 runs the device GMRES
kernels outside the conditional graph (visible to the sanitizer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

p = problems.c2_structured_3d(16)
prm = dict(problems.setup_params(2), coarse_size_target=200)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
h = airg.setup(a, **prm)
r = airg.richardson_solve(h, p.b, coarse_iterations=3)
g = airg.gmres_solve(h, p.b, coarse_iterations=3)
rf = airg.richardson_solve(h, p.b, coarse_iterations=3, fast=1)
gf = airg.gmres_solve(h, p.b, coarse_iterations=3, fast=1)
lab, _, rep = airg.cf_split(a, 0.5, 3, 0)
dl, _ = airg.dist_cf_split(a, 3)
h3 = airg.setup(a, nranks=3, **prm)
d = airg.Dist(h, 3)
rd = d.solve(p.b, coarse_iterations=3)
gd = d.solve(p.b, coarse_iterations=3, outer=1)
print("ok", r.stats.iterations, g.stats.iterations, rf.stats.iterations, gf.stats.iterations,
      rd.stats.iterations, gd.stats.iterations, int(np.array_equal(dl, lab)))
