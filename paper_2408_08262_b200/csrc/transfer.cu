// Grid-transfer operators (reference: proj/src/air.cpp:154-238).
#include "rowsplit.cuh"
#include "sparse.cuh"

namespace airg {

namespace {

__global__ void r_count(int nc, const int32_t* __restrict__ zrp, int32_t* __restrict__ cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) cnt[c] = zrp[c + 1] - zrp[c] + 1;
}

// R row c = sorted{(f_to_fine[z_col], -z), (c_to_fine[c], 1.0)}; f_to_fine
// is increasing, so the mapped Z columns stay sorted and the identity entry
// is merged in at its place (air.cpp:308-325).
__global__ void r_fill(int nc, const int32_t* __restrict__ zrp, const int32_t* __restrict__ zci,
                       const double* __restrict__ zv, const int32_t* __restrict__ f2f,
                       const int32_t* __restrict__ c2f, const int32_t* __restrict__ rrp,
                       int32_t* __restrict__ rci, double* __restrict__ rv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const int self = c2f[c];
  int o = rrp[c];
  bool placed = false;
  for (int k = zrp[c]; k < zrp[c + 1]; ++k) {
    const int col = f2f ? f2f[zci[k]] : zci[k];
    if (!placed && self < col) {
      rci[o] = self;
      rv[o++] = 1.0;
      placed = true;
    }
    rci[o] = col;
    rv[o++] = -zv[k];
  }
  if (!placed) {
    rci[o] = self;
    rv[o] = 1.0;
  }
}

// one-point prolongation (air.cpp:191-238)
// rows of a slab: local row r is global row rb + r (label / f2s are global)
__global__ void p_map(int n, const uint8_t* __restrict__ label, const int32_t* __restrict__ f2s,
                      const int32_t* __restrict__ srp, const int32_t* __restrict__ sci,
                      const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                      const double* __restrict__ av, int32_t* __restrict__ pmap, int rb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = rb + r;
  if (label[i] == AIRG_C) {
    pmap[r] = f2s[i];
    return;
  }
  int best = -1;
  double best_mag = -1.0;
  // strong C neighbours: S_i is a sorted subset of A's row -> merge walk
  int k = arp[r];
  const int ke = arp[r + 1];
  for (int t = srp[r]; t < srp[r + 1]; ++t) {
    const int j = sci[t];
    while (k < ke && aci[k] < j) ++k;
    if (label[j] != AIRG_C) continue;
    const double mag = (k < ke && aci[k] == j) ? fabs(av[k]) : 0.0;
    if (mag > best_mag) {
      best_mag = mag;
      best = j;
    }
  }
  if (best < 0) {
    for (int q = arp[r]; q < ke; ++q) {
      const int cc = aci[q];
      if (cc == i || label[cc] != AIRG_C) continue;
      const double mag = fabs(av[q]);
      if (mag > best_mag) {
        best_mag = mag;
        best = cc;
      }
    }
  }
  pmap[r] = best >= 0 ? f2s[best] : -1;
}

// The same map with S_i re-derived from A's row (coarsening.cpp:83-105: j != i,
// |a_ij| > 0, |a_ij| >= alpha * max_{k != i} |a_ik|, the product rounded once):
// S_i is A's row filtered in column order, so the strong pass visits the
// same candidates in the same order as p_map -- no S needed.
__global__ void p_map_fused(int n, const uint8_t* __restrict__ label, const int32_t* __restrict__ f2s,
                            const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                            const double* __restrict__ av, double alpha, int32_t* __restrict__ pmap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (label[i] == AIRG_C) {
    pmap[i] = f2s[i];
    return;
  }
  const int s = arp[i], e = arp[i + 1];
  double off_max = 0.0;
  for (int k = s; k < e; ++k)
    if (aci[k] != i) off_max = fmax(off_max, fabs(av[k]));
  const double thr = __dmul_rn(alpha, off_max);
  int best = -1;
  double best_mag = -1.0;
  for (int k = s; k < e; ++k) {
    const int j = aci[k];
    const double mag = fabs(av[k]);
    if (j == i || !(mag > 0.0) || !(mag >= thr) || label[j] != AIRG_C) continue;
    if (mag > best_mag) {
      best_mag = mag;
      best = j;
    }
  }
  if (best < 0) {
    for (int k = s; k < e; ++k) {
      const int j = aci[k];
      if (j == i || label[j] != AIRG_C) continue;
      const double mag = fabs(av[k]);
      if (mag > best_mag) {
        best_mag = mag;
        best = j;
      }
    }
  }
  pmap[i] = best >= 0 ? f2s[best] : -1;
}

__global__ void p_count(int n, const int32_t* __restrict__ pmap, int32_t* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cnt[i] = pmap[i] >= 0;
}
__global__ void p_fill(int n, const int32_t* __restrict__ pmap, const int32_t* __restrict__ prp,
                       int32_t* __restrict__ pci, double* __restrict__ pv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && pmap[i] >= 0) {
    pci[prp[i]] = pmap[i];
    pv[prp[i]] = 1.0;
  }
}

}  // namespace

void build_restriction(Ctx& c, const Csr& acf, const Csr& ffinv, double drop, const LabelMap& map,
                       Csr& r, const int32_t* bmap, int cb, const RowSplit* rs) {
  Csr z;
  if (rs)
    split_spgemm(c, *rs, acf, ffinv, z, drop, /*keep_diag=*/false);  // air.cpp:298-299
  else
    spgemm(c, acf, ffinv, z, drop, /*keep_diag=*/false, bmap);
  restriction_from_z(c, z, map.f_to_fine.p, map.c_to_fine.p + cb, map.n, r);
}

void restriction_from_z(Ctx& c, const Csr& z, const int32_t* f2f, const int32_t* c2f, int64_t ncols, Csr& r) {
  const int nc = z.n;
  Csr out;
  out.n = nc;
  out.m = (int32_t)ncols;
  out.rp.alloc(c, (size_t)nc + 1);
  DBuf<int32_t> cnt(c, (size_t)std::max(1, nc));
  if (nc) LAUNCH(c, r_count, blocks_for(nc, 256), 256, 0, nc, z.rp.p, cnt.p);
  out.nnz = nc ? exclusive_scan(c, cnt.p, out.rp.p, nc) : 0;
  if (!nc) CUDA_CHECK(cudaMemsetAsync(out.rp.p, 0, sizeof(int32_t), c.stream));
  out.ci.alloc(c, (size_t)out.nnz);
  out.v.alloc(c, (size_t)out.nnz);
  if (nc)
    LAUNCH(c, r_fill, blocks_for(nc, 256), 256, 0, nc, z.rp.p, z.ci.p, z.v.p, f2f, c2f, out.rp.p, out.ci.p,
           out.v.p);
  r = std::move(out);
}

void prolongation_map_fused(Ctx& c, const uint8_t* label, const int32_t* f2s, const Csr& a, double alpha,
                            int32_t* pmap) {
  if (a.n)
    LAUNCH(c, p_map_fused, blocks_for(a.n, 256), 256, 0, a.n, label, f2s, a.rp.p, a.ci.p, a.v.p, alpha, pmap);
}

void prolongation_map_rows(Ctx& c, const LabelMap& map, const Strength& g, const Csr& a, int rb,
                           int32_t* pmap) {
  if (a.n)
    LAUNCH(c, p_map, blocks_for(a.n, 256), 256, 0, a.n, map.label.p, map.fine_to_sub.p, g.rp.p, g.ci.p,
           a.rp.p, a.ci.p, a.v.p, pmap, rb);
}

void prolongation_from_map(Ctx& c, const int32_t* pmap, int n, int nc, Csr& p) {
  Csr out;
  out.n = n;
  out.m = nc;
  out.rp.alloc(c, (size_t)n + 1);
  DBuf<int32_t> cnt(c, (size_t)std::max(1, n));
  if (n) LAUNCH(c, p_count, blocks_for(n, 256), 256, 0, n, pmap, cnt.p);
  out.nnz = exclusive_scan(c, cnt.p, out.rp.p, n);
  out.ci.alloc(c, (size_t)out.nnz);
  out.v.alloc(c, (size_t)out.nnz);
  if (n) LAUNCH(c, p_fill, blocks_for(n, 256), 256, 0, n, pmap, out.rp.p, out.ci.p, out.v.p);
  p = std::move(out);
}

void build_prolongation_fused(Ctx& c, const LabelMap& map, const Csr& a, double alpha, DBuf<int32_t>& pmap,
                              Csr& p) {
  const int n = map.n;
  pmap.alloc(c, (size_t)std::max(1, n));
  if (n)
    LAUNCH(c, p_map_fused, blocks_for(n, 256), 256, 0, n, map.label.p, map.fine_to_sub.p, a.rp.p, a.ci.p, a.v.p,
           alpha, pmap.p);
  prolongation_from_map(c, pmap.p, n, map.nc, p);
}

void build_prolongation(Ctx& c, const LabelMap& map, const Strength& g, const Csr& a,
                        DBuf<int32_t>& pmap, Csr& p) {
  const int n = map.n;
  pmap.alloc(c, (size_t)n);
  prolongation_map_rows(c, map, g, a, 0, pmap.p);
  prolongation_from_map(c, pmap.p, n, map.nc, p);
}

}  // namespace airg
