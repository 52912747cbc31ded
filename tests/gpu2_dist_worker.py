"""Worker of tests/test_gpu_dist.py::test_two_process_nccl_and_p2p_match_one_gpu
(launched by torch.distributed.run, one process per GPU): the distributed
Richardson and GMRES solves over NCCL (or, with AIRG_TRANSPORT=p2p, NVLink
peer stores) against the one-GPU bits / tolerance."""
import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = airg.Context(local)
    p = problems.c2_structured_3d(32)
    prm = dict(problems.setup_params(2), coarse_size_target=500)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
    ref = airg.richardson_solve(h, p.b, coarse_iterations=3)
    refg = airg.gmres_solve(h, p.b, coarse_iterations=3)
    uid = [airg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = airg.NcclComm(ws, rank, uid[0])
    starts = np.linspace(0, p.n, ws + 1).astype(np.int64)
    d = airg.Dist(h, ws, rank=rank, comm=comm, threshold=2.0, starts=starts)
    lo, hi = starts[rank], starts[rank + 1]
    tb = ctx.to_device(p.b[lo:hi].copy())
    tx = ctx.empty(int(hi - lo), torch.float64)
    ok = True
    for _ in range(2):  # two consecutive solves (the p2p counters carry over)
        st, _ = d.solve_device(tb, tx, coarse_iterations=3)
        x = ctx.to_host(tx)
        ok &= st.iterations == ref.stats.iterations and np.array_equal(x.view(np.uint64), ref.x[lo:hi].view(np.uint64))
    st, _ = d.solve_device(tb, tx, coarse_iterations=3, outer=1)
    x = ctx.to_host(tx)
    ok &= abs(st.iterations - refg.stats.iterations) <= 1
    ok &= np.linalg.norm(x - refg.x[lo:hi]) <= 1e-8 * np.linalg.norm(refg.x)
    # owned-row setup over NCCL: this rank's rows only (global columns); the
    # hierarchy report equals the one-GPU setup's and the solve its bits
    a_loc = airg.SparseMatrix.from_arrays(int(hi - lo), p.n, p.row_offsets[lo:hi + 1] - p.row_offsets[lo],
                                          p.cols[p.row_offsets[lo]:p.row_offsets[hi]],
                                          p.vals[p.row_offsets[lo]:p.row_offsets[hi]])
    do = airg.Dist.setup_owned(airg.DeviceCSR.upload(a_loc, ctx), ws, rank=rank, comm=comm, threshold=2.0,
                               starts=starts, ctx=ctx, **prm)
    ok &= do.n_levels == h.n_levels
    for l in range(h.n_levels):
        e, o = h.level(l), do.report(l)
        ok &= (e.n, e.nnz, e.n_f, e.nnz_ffinv, e.nnz_r, e.poly_attempts) == (o.n, o.nnz, o.n_f, o.nnz_ffinv, o.nnz_r,
                                                                            o.poly_attempts)
        ok &= np.array_equal(np.array(e.coefficients), np.array(o.coefficients))
    st, _ = do.solve_device(tb, tx, coarse_iterations=3)
    x = ctx.to_host(tx)
    ok &= st.iterations == ref.stats.iterations and np.array_equal(x.view(np.uint64), ref.x[lo:hi].view(np.uint64))
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("RESULT", int(flag.item()), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
