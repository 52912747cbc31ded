import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2408_08262_b200 import airg, problems
ctx = airg.Context(0)
p = problems.make(2); prm = problems.setup_params(2)
a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
dA = airg.DeviceCSR.upload(a, ctx)
h = airg.setup(dA, ctx=ctx, **prm)
for rep in range(3):
    tot = 0; per = []
    for l in range(h.n_levels):
        Al = h.matrix_handle(l, 0); n = Al.dims()[0]
        seed = int(problems.mix(np.uint64(0), np.uint64(l)))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        airg.dist_cf_split_device(Al, [0, n], rank=-1, seed=seed, ctx=ctx)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        tot += dt; per.append(round(dt * 1e3, 2))
    print('dist P=1 emul total ms', round(tot * 1e3, 2), per[:6], per[-3:])
for rep in range(2):
    tot = 0
    for l in range(h.n_levels):
        Al = h.matrix_handle(l, 0)
        seed = int(problems.mix(np.uint64(0), np.uint64(l)))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        airg.cf_split_device(Al, 0.5, 3, seed, ctx=ctx)
        torch.cuda.synchronize(); tot += time.perf_counter() - t0
    print('fused single total ms', round(tot * 1e3, 2))
