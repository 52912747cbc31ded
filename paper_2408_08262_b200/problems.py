"""Deterministic generators for the five BASELINE.json operators (C0-C4).

The reference ships no generator for any of them: its
transport.cpp only builds the 4-angle SUPG desk operator. These generators
produce the SAME CSR bytes and right-hand side for the GPU path, the CPU
oracle and the reference arm, from the reference's counter RNG
(rng.hpp:13-29: splitmix64 / mix / uniform01) with new stream tags.

All operators are first-order upwind streaming (transport in the streaming
limit): row K has diagonal  sum_{outflow faces} (Omega.n)|f| + sigma_t |K|
and, for each inflow face shared with a neighbour N, the off-diagonal
(Omega.n)|f| < 0 in column N; inflow boundary faces carry the zero inflow
condition and are omitted. Column indices are sorted per row, int64
offsets/columns and fp64 values, i.e. the reference's SparseMatrix layout
(sparse.hpp:89-93).

Data: synthetic, seeded (seed 0 for every config unless overridden).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Counter RNG restated from rng.hpp:13-29 (vectorised, uint64 wrap-around).
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

# Stream tags for the generators (new; rng.hpp:43-46 holds the reference's).
TAG_RHS = 0x52485321     # right-hand side
TAG_OMEGA = 0x4F4D4547   # direction
TAG_SIGMA = 0x53494754   # cross sections
TAG_JITTER = 0x4A495454  # lattice jitter
TAG_DIAG = 0x44494147    # quad diagonal choice
TAG_BOXES = 0x424F5845   # C2 box partition


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> np.uint64(30))) * _C1
        x = (x ^ (x >> np.uint64(27))) * _C2
    return x ^ (x >> np.uint64(31))


def mix(seed, key):
    return splitmix64(np.asarray(seed, dtype=np.uint64) ^ splitmix64(key))


def uniform01(seed, index):
    """rng::uniform01 (rng.hpp:27-29): 53-bit mantissa in [0, 1)."""
    return (mix(seed, index) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def stream(seed: int, tag: int) -> np.uint64:
    return mix(np.uint64(seed), np.uint64(tag))


# ---------------------------------------------------------------------------
@dataclass
class Problem:
    name: str
    n: int
    row_offsets: np.ndarray  # int64 [n+1]
    cols: np.ndarray         # int64 [nnz]
    vals: np.ndarray         # float64 [nnz]
    b: np.ndarray            # float64 [n]
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])


def _csr_from_coo(n: int, rows, cols, vals) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Sorted CSR; duplicate (row, col) pairs are summed in sorted order,
    as SparseMatrix::from_triplets (sparse.cpp:48-80)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    key = rows * np.int64(n) + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    summed = np.add.reduceat(vals, start) if len(vals) else vals
    r = uniq // n
    c = uniq % n
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(offsets, r + 1, 1)
    return np.cumsum(offsets), c.astype(np.int64), summed


def _rhs(n: int, seed: int) -> np.ndarray:
    return uniform01(stream(seed, TAG_RHS), np.arange(n, dtype=np.uint64))


# ---------------------------------------------------------------------------
def c0_structured_2d(nx: int = 128, angle: float = 0.3, sigma_t: float = 0.0,
                     seed: int = 0) -> Problem:
    """BASELINE config 0: 2D structured upwind, Omega = (cos a, sin a),
    diagonal |Ox|/h + |Oy|/h + sigma_t, upwind neighbours -|Ox|/h, -|Oy|/h,
    h = 1/nx, zero inflow. Cell (i, j) is row j*nx + i."""
    h = 1.0 / nx
    ox, oy = math.cos(angle), math.sin(angle)
    return _structured(nx, (ox, oy), h, np.full(nx * nx, sigma_t), seed, "C0", dims=2)


def c2_structured_3d(nx: int = 128, seed: int = 0, nz_slabs: int = 1) -> Problem:
    """BASELINE config 2: 3D structured 7-point upwind, 128^3 cells, seed-random
    unit Omega, sigma_t piecewise constant over 8 random boxes in [0, 1e-2]
    (the cube split by one random plane per axis, positions U[0.25, 0.75]).
    nz_slabs > 1 stacks that many nx^3 cubes along z (nx x nx x nz_slabs*nx
    cells, h = 1/nx): the weak-scaling family, one z-slab per GPU."""
    if nz_slabs > 1:
        return _c2_stacked(nx, seed, nz_slabs)
    s_om = stream(seed, TAG_OMEGA)
    g = np.array([_normal(s_om, k) for k in range(3)])
    om = g / np.linalg.norm(g)
    s_box = stream(seed, TAG_BOXES)
    cuts = 0.25 + 0.5 * uniform01(s_box, np.arange(3, dtype=np.uint64))
    sig_box = 1e-2 * uniform01(stream(seed, TAG_SIGMA), np.arange(8, dtype=np.uint64))
    h = 1.0 / nx
    c = (np.arange(nx) + 0.5) * h
    bx = (c >= cuts[0]).astype(np.int64)
    by = (c >= cuts[1]).astype(np.int64)
    bz = (c >= cuts[2]).astype(np.int64)
    box = (bz[:, None, None] * 4 + by[None, :, None] * 2 + bx[None, None, :]).ravel()
    p = _structured(nx, tuple(om), h, sig_box[box], seed, "C2", dims=3)
    p.meta.update(omega=om.tolist(), cuts=cuts.tolist(), sigma_boxes=sig_box.tolist())
    return p


def _c2_stacked(nx: int, seed: int, slabs: int) -> Problem:
    """C2 operator on nx x nx x (slabs*nx) cells: the same Omega and box
    cross sections repeated per stacked cube (weak scaling in z)."""
    s_om = stream(seed, TAG_OMEGA)
    g = np.array([_normal(s_om, k) for k in range(3)])
    om = g / np.linalg.norm(g)
    s_box = stream(seed, TAG_BOXES)
    cuts = 0.25 + 0.5 * uniform01(s_box, np.arange(3, dtype=np.uint64))
    sig_box = 1e-2 * uniform01(stream(seed, TAG_SIGMA), np.arange(8, dtype=np.uint64))
    h = 1.0 / nx
    c = (np.arange(nx) + 0.5) * h
    bx = (c >= cuts[0]).astype(np.int64)
    by = (c >= cuts[1]).astype(np.int64)
    bz = np.tile((c >= cuts[2]).astype(np.int64), slabs)
    box = (bz[:, None, None] * 4 + by[None, :, None] * 2 + bx[None, None, :]).ravel()
    nz = slabs * nx
    n = nx * nx * nz
    idx = np.arange(n, dtype=np.int64)
    coord = [idx % nx, (idx // nx) % nx, idx // (nx * nx)]
    dims_n = [nx, nx, nz]
    strides = [1, nx, nx * nx]
    rows, cols, vals = [idx], [idx], [sum(abs(o) for o in om) / h + sig_box[box]]
    for d in range(3):
        step = -1 if om[d] > 0 else 1
        ok = (coord[d] + step >= 0) & (coord[d] + step < dims_n[d])
        r = idx[ok]
        rows.append(r)
        cols.append(r + step * strides[d])
        vals.append(np.full(r.size, -abs(om[d]) / h))
    ro, co, va = _csr_from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    return Problem("C2x%d" % slabs, n, ro, co, va, _rhs(n, seed),
                   dict(nx=nx, nz=nz, slabs=slabs, omega=om.tolist(), h=h))


def _normal(seed, index: int) -> float:
    """rng::standard_normal (rng.hpp:32-39), Box-Muller."""
    u1 = (float(mix(seed, np.uint64(2 * index)) >> np.uint64(11)) + 1.0) * 2.0 ** -53
    u2 = float(mix(seed, np.uint64(2 * index + 1)) >> np.uint64(11)) * 2.0 ** -53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def _structured(nx: int, om, h: float, sigma: np.ndarray, seed: int, name: str,
                dims: int) -> Problem:
    n = nx ** dims
    idx = np.arange(n, dtype=np.int64)
    coord = [(idx // nx ** d) % nx for d in range(dims)]  # d=0 fastest (x)
    diag = sum(abs(o) for o in om) / h + sigma
    rows = [idx]
    cols = [idx]
    vals = [diag]
    for d in range(dims):
        if om[d] == 0.0:
            continue
        step = -1 if om[d] > 0 else 1      # upwind neighbour along axis d
        ok = (coord[d] + step >= 0) & (coord[d] + step < nx)
        r = idx[ok]
        rows.append(r)
        cols.append(r + step * nx ** d)
        vals.append(np.full(r.size, -abs(om[d]) / h))
    ro, co, va = _csr_from_coo(n, np.concatenate(rows), np.concatenate(cols),
                               np.concatenate(vals))
    return Problem(name, n, ro, co, va, _rhs(n, seed),
                   dict(nx=nx, dims=dims, omega=list(om), h=h))


# ---------------------------------------------------------------------------
def _tri_lattice(nx: int, jitter: float, seed: int):
    """(nx+1)^2 lattice on [0,1]^2, interior points jittered by U[-j, j] h,
    each quad split along a seed-random diagonal; triangles CCW, quad-major
    order (2 per quad)."""
    h = 1.0 / nx
    m = nx + 1
    ids = np.arange(m * m, dtype=np.int64)
    ix, iy = ids % m, ids // m
    sj = stream(seed, TAG_JITTER)
    u0 = 2.0 * uniform01(sj, (2 * ids).astype(np.uint64)) - 1.0
    u1 = 2.0 * uniform01(sj, (2 * ids + 1).astype(np.uint64)) - 1.0
    interior = (ix > 0) & (ix < nx) & (iy > 0) & (iy < nx)
    x = ix * h + np.where(interior, jitter * h * u0, 0.0)
    y = iy * h + np.where(interior, jitter * h * u1, 0.0)
    q = np.arange(nx * nx, dtype=np.int64)
    qx, qy = q % nx, q // nx
    n00 = qy * m + qx
    n10, n01, n11 = n00 + 1, n00 + m, n00 + m + 1
    flip = uniform01(stream(seed, TAG_DIAG), q.astype(np.uint64)) < 0.5
    t0 = np.where(flip[:, None], np.stack([n00, n10, n11], 1), np.stack([n00, n10, n01], 1))
    t1 = np.where(flip[:, None], np.stack([n00, n11, n01], 1), np.stack([n10, n11, n01], 1))
    tris = np.stack([t0, t1], 1).reshape(-1, 3)
    return np.stack([x, y], 1), tris


def _upwind_fv_2d(pts: np.ndarray, tris: np.ndarray, om, sigma: np.ndarray):
    """P0 upwind finite volume: rows/cols/vals for one angle block."""
    nt = len(tris)
    p = pts[tris]                                   # [nt, 3, 2]
    area = 0.5 * ((p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1])
                  - (p[:, 2, 0] - p[:, 0, 0]) * (p[:, 1, 1] - p[:, 0, 1]))
    a = tris
    b = np.roll(tris, -1, axis=1)
    pa, pb = pts[a], pts[b]                          # [nt, 3, 2]
    dx, dy = pb[..., 0] - pa[..., 0], pb[..., 1] - pa[..., 1]
    flux = om[0] * dy - om[1] * dx                   # (Omega . n_out)|e| (CCW)
    lo, hi = np.minimum(a, b).ravel(), np.maximum(a, b).ravel()
    key = lo * (pts.shape[0] + 1) + hi
    cell = np.repeat(np.arange(nt, dtype=np.int64), 3)
    order = np.argsort(key, kind="stable")
    ks = key[order]
    same = ks[1:] == ks[:-1]
    nbr = np.full(3 * nt, -1, dtype=np.int64)
    i0, i1 = order[:-1][same], order[1:][same]
    nbr[i0] = cell[i1]
    nbr[i1] = cell[i0]
    f = flux.ravel()
    diag = np.zeros(nt)
    np.add.at(diag, cell[f > 0], f[f > 0])
    diag += sigma * area
    inflow = (f < 0) & (nbr >= 0)
    rows = np.concatenate([np.arange(nt, dtype=np.int64), cell[inflow]])
    cols = np.concatenate([np.arange(nt, dtype=np.int64), nbr[inflow]])
    vals = np.concatenate([diag, f[inflow]])
    return rows, cols, vals, area


def c1_unstructured_2d(nx: int = 512, seed: int = 0, sigma_max: float = 1e-3,
                       angle: float | None = None, jitter: float = 0.25) -> Problem:
    """BASELINE config 1: 2D unstructured P0 upwind FV on a jittered nx^2
    lattice (2 nx^2 triangles), one seed-random direction angle in [0, 2pi),
    sigma_t ~ U[0, sigma_max] per cell."""
    pts, tris = _tri_lattice(nx, jitter, seed)
    if angle is None:
        angle = 2.0 * math.pi * float(uniform01(stream(seed, TAG_OMEGA), np.uint64(0)))
    nt = len(tris)
    sig = sigma_max * uniform01(stream(seed, TAG_SIGMA), np.arange(nt, dtype=np.uint64))
    rows, cols, vals, _ = _upwind_fv_2d(pts, tris, (math.cos(angle), math.sin(angle)), sig)
    ro, co, va = _csr_from_coo(nt, rows, cols, vals)
    return Problem("C1", nt, ro, co, va, _rhs(nt, seed), dict(nx=nx, angle=angle))


def c3_sn_2d(nx: int = 256, n_angles: int = 64, seed: int = 0) -> Problem:
    """BASELINE config 3: the C1-style operator on nx^2 jittered quads
    (2 nx^2 triangles) for each of n_angles ordinates theta_k = 2 pi k / n,
    block diagonal (angle-major rows), sigma_t = 0."""
    pts, tris = _tri_lattice(nx, 0.25, seed)
    nt = len(tris)
    ro_all, co_all, va_all = [np.zeros(1, dtype=np.int64)], [], []
    base = 0
    for k in range(n_angles):
        th = 2.0 * math.pi * k / n_angles
        rows, cols, vals, _ = _upwind_fv_2d(pts, tris, (math.cos(th), math.sin(th)), np.zeros(nt))
        ro, co, va = _csr_from_coo(nt, rows, cols, vals)
        ro_all.append(ro[1:] + ro_all[-1][-1])
        co_all.append(co + base)
        va_all.append(va)
        base += nt
    n = nt * n_angles
    return Problem("C3", n, np.concatenate(ro_all), np.concatenate(co_all),
                   np.concatenate(va_all), _rhs(n, seed),
                   dict(nx=nx, n_angles=n_angles, block=nt))


# ---------------------------------------------------------------------------
# Kuhn (Freudenthal) split of a cube into 6 tetrahedra sharing the main
# diagonal v0 -> v7; conforming across cubes with one orientation.
_KUHN = np.array([[0, 1, 3, 7], [0, 1, 5, 7], [0, 2, 3, 7],
                  [0, 2, 6, 7], [0, 4, 5, 7], [0, 4, 6, 7]])


def c4_tets_3d(nx: int = 70, ny: int = 70, nz: int = 68, seed: int = 0,
               jitter: float = 0.2, sigma_max: float = 1e-3, z0: int = 0,
               nz_total: int | None = None) -> Problem:
    """BASELINE config 4: jittered cube lattice (+-0.2h), 6 tets per cube,
    P0 upwind flux (Omega.n)|face|, seed-random Omega, sigma_t ~ U[0,1e-3].
    Default 70 x 70 x 68 cubes = 1,999,200 tets (the 2M-per-GPU slab);
    z-slab partition: rank r owns cube layers [68 r, 68 (r+1)).  z0/nz_total
    select a slab of a taller global lattice (global ids, weak scaling)."""
    nz_total = nz if nz_total is None else nz_total
    h = 1.0 / max(nx, ny)
    mx, my, mz = nx + 1, ny + 1, nz_total + 1
    # lattice points of this slab (+ one layer above/below for neighbours)
    zlo, zhi = max(z0 - 1, 0), min(z0 + nz + 1, nz_total)
    pid = np.arange(mx * my * mz, dtype=np.int64).reshape(mz, my, mx)[zlo:zhi + 1].ravel()
    ix, iy, iz = pid % mx, (pid // mx) % my, pid // (mx * my)
    sj = stream(seed, TAG_JITTER)
    interior = (ix > 0) & (ix < nx) & (iy > 0) & (iy < ny) & (iz > 0) & (iz < nz_total)
    jit = [np.where(interior, jitter * h * (2.0 * uniform01(sj, (3 * pid + d).astype(np.uint64)) - 1.0), 0.0)
           for d in range(3)]
    pts = np.zeros((mx * my * mz, 3))
    pts[pid, 0] = ix * h + jit[0]
    pts[pid, 1] = iy * h + jit[1]
    pts[pid, 2] = iz * h + jit[2]
    # cubes of layers [zlo, zhi) -> tets; global tet id = cube_id*6 + k
    cz, cy, cx = np.meshgrid(np.arange(zlo, zhi), np.arange(ny), np.arange(nx), indexing="ij")
    cz, cy, cx = cz.ravel(), cy.ravel(), cx.ravel()
    corner = np.stack([((cz + (v >> 2 & 1)) * my + cy + (v >> 1 & 1)) * mx + cx + (v & 1)
                       for v in range(8)], 1)
    tets = corner[:, _KUHN].reshape(-1, 4)
    cube_ids = (cz * ny + cy) * nx + cx
    gid = (cube_ids[:, None] * 6 + np.arange(6)).ravel()
    s_om = stream(seed, TAG_OMEGA)
    g = np.array([_normal(s_om, k) for k in range(3)])
    om = g / np.linalg.norm(g)
    own = (gid >= z0 * nx * ny * 6) & (gid < (z0 + nz) * nx * ny * 6)
    # faces: opposite vertex k -> face of the other three
    faces = np.stack([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]], tets[:, [0, 1, 2]]], 1)
    opp = tets
    P = pts[faces]                                   # [nt, 4, 3, 3]
    nrm = 0.5 * np.cross(P[:, :, 1] - P[:, :, 0], P[:, :, 2] - P[:, :, 0])  # area-weighted
    out = np.einsum("tfd,tfd->tf", nrm, P[:, :, 0] - pts[opp])
    nrm = np.where((out > 0)[..., None], nrm, -nrm)
    flux = nrm @ om                                  # (Omega . n_out)|f|
    vol = np.abs(np.einsum("td,td->t", pts[tets[:, 1]] - pts[tets[:, 0]],
                           np.cross(pts[tets[:, 2]] - pts[tets[:, 0]], pts[tets[:, 3]] - pts[tets[:, 0]]))) / 6.0
    fs = np.sort(faces, axis=2).reshape(-1, 3)
    M = np.int64(mx * my * mz + 1)
    key = (fs[:, 0] * M + fs[:, 1]) * M + fs[:, 2]
    cell = np.repeat(gid, 4)
    order = np.argsort(key, kind="stable")
    ks = key[order]
    same = ks[1:] == ks[:-1]
    nbr = np.full(len(key), -1, dtype=np.int64)
    i0, i1 = order[:-1][same], order[1:][same]
    nbr[i0] = cell[i1]
    nbr[i1] = cell[i0]
    f = flux.ravel()
    nt_all = len(tets)
    sig = sigma_max * uniform01(stream(seed, TAG_SIGMA), gid.astype(np.uint64))
    loc = np.repeat(np.arange(nt_all), 4)
    diag = np.zeros(nt_all)
    np.add.at(diag, loc[f > 0], f[f > 0])
    diag += sig * vol
    inflow = (f < 0) & (nbr >= 0)
    own_f = np.repeat(own, 4)
    base = z0 * nx * ny * 6
    rows = np.concatenate([gid[own] - base, cell[inflow & own_f] - base])
    cols = np.concatenate([gid[own], nbr[inflow & own_f]])
    vals = np.concatenate([diag[own], f[inflow & own_f]])
    n = int(own.sum())
    # columns stay global (slab halo columns < base or >= base + n)
    ncols = nx * ny * nz_total * 6
    key2 = rows * np.int64(ncols) + cols
    o2 = np.argsort(key2, kind="stable")
    rows, cols, vals = rows[o2], cols[o2], vals[o2]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(offsets, rows + 1, 1)
    offsets = np.cumsum(offsets)
    b = uniform01(stream(seed, TAG_RHS), gid[own].astype(np.uint64))
    return Problem("C4", n, offsets, cols.astype(np.int64), vals, b,
                   dict(nx=nx, ny=ny, nz=nz, z0=z0, nz_total=nz_total, omega=om.tolist(),
                        global_cols=ncols, row_base=base))


def make(config: int, scale: float = 1.0, seed: int = 0) -> Problem:
    """Config index (BASELINE.json configs[i]); scale < 1 shrinks the grid
    (for oracle-sized parity cases) keeping the construction."""
    def s(n):
        return max(4, int(round(n * scale)))
    if config == 0:
        return c0_structured_2d(s(128), seed=seed)
    if config == 1:
        return c1_unstructured_2d(s(512), seed=seed)
    if config == 2:
        return c2_structured_3d(s(128), seed=seed)
    if config == 3:
        return c3_sn_2d(s(256), n_angles=64 if scale >= 1 else max(2, int(64 * scale)), seed=seed)
    if config == 4:
        return c4_tets_3d(s(70), s(70), s(68), seed=seed)
    raise ValueError(f"unknown config {config}")


# AIRG parameters per config (BASELINE.json): alpha 0.5, DDC 0.1,
# poly order 4, sparsity 1; C0-C1 keep the reference truncation defaults
# (3000 rows, coarse order 12); C2-C4 truncate at 5000 with coarse order 8.
def setup_params(config: int) -> dict:
    p = dict(strength_alpha=0.5, ddc_fraction=0.1, ddc_bins=1000, max_loops=3,
             poly_order=4, sparsity_order=1, drop_coarse=0.001, drop_restrict=0.01,
             coarse_size_target=3000, coarse_poly_order=12, coarse_iterations=3, seed=0)
    if config >= 2:
        p.update(coarse_size_target=5000, coarse_poly_order=8)
    return p


def gather_csr_slabs(ps: Problem, world: int, all_gather) -> tuple[int, np.ndarray, np.ndarray, np.ndarray]:
    """The global CSR from every rank's row slab (rows in rank order, global
    column indices, e.g. the C4 z-slabs of c4_tets_3d(z0=..., nz_total=...)).
    all_gather(list_of_world_tensors, tensor) is torch.distributed.all_gather
    (any backend). Returns (N, row_offsets, cols, vals) as numpy arrays."""
    import torch
    dev = None
    probe = torch.zeros(1)
    try:  # NCCL gathers device tensors; gloo host tensors
        import torch.distributed as dist
        if dist.is_initialized() and dist.get_backend() == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
    except Exception:
        dev = None
    mk = (lambda t: t.to(dev)) if dev is not None else (lambda t: t)
    cnt = mk(torch.tensor([ps.nnz, ps.n], dtype=torch.int64))
    cnts = [mk(torch.zeros(2, dtype=torch.int64)) for _ in range(world)]
    all_gather(cnts, cnt)
    nnz = [int(c[0]) for c in cnts]
    rows = [int(c[1]) for c in cnts]
    mz, mr = max(nnz), max(rows)
    ci = mk(torch.zeros(mz, dtype=torch.int64))
    va = mk(torch.zeros(mz, dtype=torch.float64))
    rl = mk(torch.zeros(mr, dtype=torch.int64))
    ci[: ps.nnz] = mk(torch.from_numpy(np.asarray(ps.cols, np.int64)))
    va[: ps.nnz] = mk(torch.from_numpy(np.asarray(ps.vals, np.float64)))
    rl[: ps.n] = mk(torch.from_numpy(np.diff(ps.row_offsets).astype(np.int64)))
    cis = [torch.empty_like(ci) for _ in range(world)]
    vas = [torch.empty_like(va) for _ in range(world)]
    rls = [torch.empty_like(rl) for _ in range(world)]
    all_gather(cis, ci)
    all_gather(vas, va)
    all_gather(rls, rl)
    n = sum(rows)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(np.concatenate([rls[r][: rows[r]].cpu().numpy() for r in range(world)]))
    cols = np.concatenate([cis[r][: nnz[r]].cpu().numpy() for r in range(world)])
    vals = np.concatenate([vas[r][: nnz[r]].cpu().numpy() for r in range(world)])
    return n, rp, cols, vals
