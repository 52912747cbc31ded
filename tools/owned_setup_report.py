"""Owned-row distributed setup on full-size C4 in emulation (all P ranks in
one process on one GPU): per-rank resident bytes of the distribution for
P = 1, 2, 4, 8 z-slabs, the halving schedule, and agreement of every level's
report with the single-GPU setup. Writes gpurun_out/owned_setup.txt.

  python tools/owned_setup_report.py [--scale 1.0]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

FIELDS = ("n", "nnz", "n_f", "n_c", "nnz_ff", "nnz_fc", "nnz_cf", "nnz_ffinv", "nnz_r", "nnz_p", "poly_attempts",
          "effective_order")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default="gpurun_out/owned_setup.txt")
    args = ap.parse_args()
    ctx = airg.Context(0)
    nxy = round(70 * args.scale)
    nz = round(68 * args.scale)
    p = problems.c4_tets_3d(nxy, nxy, nz)
    prm = problems.setup_params(4)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    dA = airg.DeviceCSR.upload(a, ctx)
    h = airg.setup(dA, ctx=ctx, **prm)
    lines = [f"C4 {nxy} x {nxy} x {nz} cubes x 6 = {p.n} tets, nnz {p.nnz}; single-GPU setup: {h.n_levels} levels"]
    for P in (1, 2, 4, 8):
        starts = np.linspace(0, p.n, P + 1).astype(np.int64)
        t0 = time.perf_counter()
        d = airg.Dist.setup_owned(dA, P, threshold=2.0, starts=starts, ctx=ctx, **prm)
        wall = (time.perf_counter() - t0) * 1e3
        same = d.n_levels == h.n_levels and all(
            all(getattr(h.level(l), f) == getattr(d.report(l), f) for f in FIELDS)
            and np.array_equal(np.array(h.level(l).coefficients), np.array(d.report(l).coefficients))
            for l in range(h.n_levels))
        rb = [d.rank_bytes(r) for r in range(P)]
        act = [d.level_info(l)["active"] for l in range(d.n_levels + 1)]
        lines.append(f"P={P}: reports equal to one GPU: {same}; rank bytes max {max(rb) / 1e6:.1f} MB, "
                     f"sum {sum(rb) / 1e6:.1f} MB, per rank {[round(x / 1e6, 1) for x in rb]}; "
                     f"active ranks per level {act}; emulated setup wall {wall:.0f} ms (all ranks serial)")
        del d
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
