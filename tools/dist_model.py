"""Partition report of the bench's weak-scaling system at P = 2, 4, 8 slabs,
built and partitioned on ONE GPU (airg_dist_create in emulation; nothing is
timed across ranks): per level the active ranks after the replay rule
(partition_model.cpp:77-112, threshold 2), the local / non-local nnz ratio
before and after, and the halo entries, plus a bandwidth model of one
V-cycle's halo traffic against the measured one-GPU step.

  python tools/dist_model.py > profiles/r1_dist_partition.txt   (GPU box)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_08262_b200 import airg, problems  # noqa: E402

NVLINK_GBS = 900.0  # per direction per GPU (NVLink 5 through NVSwitch)
EXCH_PER_LEVEL = 6  # R b, P e_c, first F residual, 2 x F update, second F residual

ctx = airg.Context(0)
prm = problems.setup_params(2)
for P in (2, 4, 8):
    p = problems.c2_structured_3d(128, nz_slabs=P)
    a = airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)
    h = airg.setup(airg.DeviceCSR.upload(a, ctx), ctx=ctx, **prm)
    slab = p.n // P
    starts = np.arange(P + 1, dtype=np.int64) * slab
    d = airg.Dist(h, P, rank=-1, threshold=2.0, starts=starts)
    L = h.n_levels
    print(f"P = {P}: n = {p.n:,} ({slab:,} per slab), {L} levels")
    print(f"{'lvl':>4} {'n':>10} {'active':>6} {'ratio':>8} {'ratio_after':>11} {'halo':>9} {'halo/row %':>10}")
    halo_bytes = 0
    for l in range(L):
        li = d.level_info(l)
        n_l = h.level(l).n
        halo_bytes += EXCH_PER_LEVEL * 8 * li["halo"]
        print(f"{l:4d} {n_l:10d} {li['active']:6d} {li['ratio_before']:8.2f} {li['ratio_after']:11.2f} "
              f"{li['halo']:9d} {100.0 * li['halo'] / max(n_l, 1):10.3f}{'  <- halving' if li['triggered'] else ''}")
    # each rank sends ~ its share; model the busiest link as total / active ranks of level 0
    t_us = halo_bytes / P / (NVLINK_GBS * 1e3)
    print(f"model: ~{halo_bytes / 1e6:.2f} MB of halo per V-cycle over all ranks "
          f"(~{EXCH_PER_LEVEL} exchanges per level), ~{t_us:.1f} us per rank at {NVLINK_GBS:.0f} GB/s "
          f"if not overlapped; per-exchange launch/latency floor dominates: "
          f"{EXCH_PER_LEVEL * L} exchanges per V-cycle\n")
    del d, h
