import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
import __graft_entry__ as g
g.smoke()
from paper_2408_08262_b200 import airg, problems
import refpy
for cfg, scale in [(0, 1.0), (2, 0.25), (1, 0.25), (2, 1.0)]:
    p = problems.make(cfg, scale); prm = problems.setup_params(cfg)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    orc = refpy.port()
    t=time.time(); lab, pre, rep = airg.cf_split(a, seed=0); tg=time.time()-t
    A = orc.mat_from_problem(p)
    t=time.time(); ol, op, orep = refpy.cf_split(orc, A, prm, 0); to=time.time()-t
    print(f"C{cfg}x{scale} n={p.n} cf_split labels equal={np.array_equal(lab, ol)} pre equal={np.array_equal(pre, op)} gpu {tg:.3f}s oracle {to:.3f}s rep {rep}", flush=True)
    x = np.random.default_rng(0).standard_normal(p.n)
    y = airg.spmv(a, x); yo = refpy.spmv(orc, A, x)
    print("  spmv bitwise:", np.array_equal(y.view(np.uint64), yo.view(np.uint64)), flush=True)
    t=time.time(); h = airg.setup(a, **prm); ts=time.time()-t
    info = h.info()
    print(f"  native setup {ts:.2f}s levels {info.n_levels} coarse {info.coarse_n} oc {info.operator_complexity:.3f}", flush=True)
    t=time.time(); res = airg.richardson_solve(h, p.b, coarse_iterations=prm['coarse_iterations']); tsol=time.time()-t
    print(f"  solve {tsol:.3f}s its {res.stats.iterations} rel {res.stats.final_relative_residual:.3e} inner {res.stats.solve_seconds:.4f}s", flush=True)
    resg = airg.gmres_solve(h, p.b, coarse_iterations=prm['coarse_iterations'])
    print(f"  gmres its {resg.stats.iterations} rel {resg.stats.final_relative_residual:.3e} inner {resg.stats.solve_seconds:.4f}s", flush=True)
