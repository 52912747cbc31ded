"""CPU checks of the N > 1 host logic (no GPU): the halo plan rule of the
row-slab decomposition (airg_dist_plan_host, the rule the device build
applies), exercised by two real processes over torch.distributed `gloo`
(world_size 2): each rank plans its slab, the ranks exchange requests and
halo values, and the local products over [owned | halo] reproduce the
global SpMV rows bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_08262_b200 import airg, problems


def test_plan_host_rule():
    a = problems.c0_structured_2d(32)
    starts = np.array([0, 300, 700, 1024], np.int64)
    for r in range(3):
        lo, hi = starts[r], starts[r + 1]
        cols = a.cols[a.row_offsets[lo]:a.row_offsets[hi]]
        halo, rc = airg.plan_host(starts, r, cols)
        exp = np.unique(cols[(cols < lo) | (cols >= hi)])
        assert np.array_equal(halo, exp) and rc.sum() == len(exp) and rc[r] == 0
        # receive counts grouped by owner, owners ascending
        owners = np.searchsorted(starts, halo, side="right") - 1
        assert np.array_equal(np.bincount(owners, minlength=3), rc)
    with pytest.raises(airg.InvalidArgument):
        airg.plan_host(starts, 3, a.cols[:4])
    # the p2p push rule: every receiver's halo entry is pushed by its owner,
    # once, to slot own + (its position in the receiver's sorted halo)
    for q in range(3):
        lo, hi = starts[q], starts[q + 1]
        halo, _ = airg.plan_host(starts, q, a.cols[a.row_offsets[lo]:a.row_offsets[hi]])
        filled = np.zeros(len(halo), int)
        for r in range(3):
            if r == q:
                continue
            si, pos = airg.p2p_push_plan_host(starts, r, halo, q)
            assert np.array_equal(starts[r] + si, halo[pos - (hi - lo)])
            filled[pos - (hi - lo)] += 1
        assert (filled == 1).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ordered_rows(rp, ci, v, x):
    """Reference-order row sums (sparse.cpp:193-198) in numpy loops."""
    y = np.zeros(len(rp) - 1)
    for i in range(len(rp) - 1):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc = acc + v[k] * x[ci[k]]
        y[i] = acc
    return y


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = problems.c2_structured_3d(8)          # 512 rows, 7-point upwind
        n = a.n
        starts = np.array([0, 256, 512], np.int64)  # two z-slabs
        lo, hi = starts[rank], starts[rank + 1]
        rp = a.row_offsets[lo:hi + 1] - a.row_offsets[lo]
        ci = a.cols[a.row_offsets[lo]:a.row_offsets[hi]]
        v = a.vals[a.row_offsets[lo]:a.row_offsets[hi]]
        halo, recv = airg.plan_host(starts, rank, ci)
        x_global = np.sin(np.arange(n) * 0.37)
        x_own = x_global[lo:hi].copy()
        # request lists: ship my halo to the owners (all_gather of ragged lists)
        lists = [None] * world
        dist.all_gather_object(lists, halo.tolist())
        peer = 1 - rank
        send_idx = np.array([g - lo for g in lists[peer] if lo <= g < hi], np.int64)
        sbuf = torch.from_numpy(x_own[send_idx].copy())
        rbuf = torch.zeros(int(recv[peer]), dtype=torch.float64)
        reqs = [dist.isend(sbuf, peer), dist.irecv(rbuf, peer)]
        for q in reqs:
            q.wait()
        x_local = np.concatenate([x_own, rbuf.numpy()])
        # remap columns to [owned | halo]
        loc = np.where((ci >= lo) & (ci < hi), ci - lo, hi - lo + np.searchsorted(halo, ci))
        y_local = _ordered_rows(rp, loc, v, x_local)
        y_ref = _ordered_rows(a.row_offsets, a.cols, a.vals, x_global)[lo:hi]
        ok = np.array_equal(y_local.view(np.uint64), y_ref.view(np.uint64))
        # the reference's locality ratio for this 2-slab partition (partition_model.cpp:53-64)
        local = int(((ci >= lo) & (ci < hi)).sum())
        t = torch.tensor([local, len(ci) - local], dtype=torch.int64)
        g = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(g, t)
        ratio = np.mean([int(x[0]) / int(x[1]) for x in g if int(x[1]) > 0])
        # the p2p transport's addressing (airg_p2p_push_plan_host): the peer
        # computes where each of its values lands in MY [own | halo] buffer
        # from my plan alone; ship (position, value) pairs and place them
        my_push_idx, my_push_pos = airg.p2p_push_plan_host(starts, rank, np.array(lists[peer], np.int64), peer)
        pair = torch.from_numpy(np.stack([my_push_pos.astype(np.float64), x_own[my_push_idx]]).copy())
        n_in = torch.tensor([pair.shape[1]], dtype=torch.int64)
        n_peer = torch.zeros(1, dtype=torch.int64)
        reqs = [dist.isend(n_in, peer), dist.irecv(n_peer, peer)]
        for q in reqs:
            q.wait()
        got = torch.zeros((2, int(n_peer[0])), dtype=torch.float64)
        reqs = [dist.isend(pair, peer), dist.irecv(got, peer)]
        for q in reqs:
            q.wait()
        x_p2p = np.full(hi - lo + len(halo), np.nan)
        x_p2p[: hi - lo] = x_own
        x_p2p[got[0].numpy().astype(np.int64)] = got[1].numpy()
        ok_p2p = not np.isnan(x_p2p).any() and np.array_equal(x_p2p.view(np.uint64), x_local.view(np.uint64))
        result_q.put((rank, bool(ok and ok_p2p), len(halo), float(ratio)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_halo_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok, _, _ in res), res
    # upwind streaming: the halo is one-sided (only the downwind slab needs
    # the upwind slab's boundary plane)
    assert res[0][2] + res[1][2] == 64 and min(res[0][2], res[1][2]) == 0
    assert res[0][3] == res[1][3] and res[0][3] > 2.0


def _slab_worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = problems.c4_tets_3d(6, 5, 4, z0=4 * rank, nz_total=4 * world)
        n, rp, ci, v = problems.gather_csr_slabs(ps, world, dist.all_gather)
        g = problems.c4_tets_3d(6, 5, 4 * world)
        ok = (n == g.n and np.array_equal(rp, g.row_offsets) and np.array_equal(ci, g.cols)
              and np.array_equal(v.view(np.uint64), g.vals.view(np.uint64))
              and np.array_equal(ps.b.view(np.uint64), g.b[ps.n * rank: ps.n * (rank + 1)].view(np.uint64)))
        result_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_c4_zslabs_gather_to_global_operator():
    """The weak-scaling bench's N > 1 input path (bench.py run_gpu_dist): each
    rank generates its C4 z-slab (global columns) and the all-gathered slabs
    are the global operator and right-hand side, bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok in res), res
