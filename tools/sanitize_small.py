"""Small end-to-end run for compute-sanitizer (memcheck / racecheck): setup,
CF split, Richardson and GMRES solves, distributed emulation, Matrix Market."""
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
lab, _, rep = airg.cf_split(a, 0.5, 3, 0)
dl, _ = airg.dist_cf_split(a, 3)
h3 = airg.setup(a, nranks=3, **prm)
d = airg.Dist(h, 3)
rd = d.solve(p.b, coarse_iterations=3)
print("ok", r.stats.iterations, g.stats.iterations, rd.stats.iterations, int(np.array_equal(dl, lab)))
