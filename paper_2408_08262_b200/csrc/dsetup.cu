// Owned-row distributed AIRG setup (SURVEY §8e "setup collectives", §8f-3).
//
// The reference's setup (air.cpp:285-434) level by level, every rank holding
// and building only ITS rows of every operator (no rank ever holds a whole
// level operator; the coarsest grid alone is gathered on rank 0):
//   A_l rows of the level partition
//   -> CF split on the slabs (dist.cu cf_split_slabs: halo exchanges and
//      allreduces, labels bit-identical to one GPU)
//   -> global F / C numbers (prefix over the ranks) exchanged for the halo
//   -> A_ff, A_fc, A_cf, A_F of the own rows
//   -> Aff^-1 by the GMRES polynomial: power basis by distributed
//      double-double SpMVs, the Gram matrix per rank summed over the ranks in
//      rank order (the same host fit on every rank), the fixed-sparsity
//      assembly of the own F rows from the A_ff halo rows gathered once
//      (PAPER.md:133), the growth guard by a distributed power iteration
//   -> Z = A_cf Aff^-1 from the Aff^-1 halo rows (distance 2), R = [Z | I]
//   -> one-point P from the exchanged coarse numbers, A P (halo P entries)
//   -> R (A P) from the A P halo rows (distance 2) = the coarse rows, moved
//      to the next level's partition (balanced, then the replay halving rule
//      of partition_model.cpp:77-112 on distributed locality counts)
//   -> ... -> the coarsest grid gathered on rank 0 for the coarse polynomial.
// Every row is produced by the one-GPU kernel on the same row with the same
// entry order, so the operators equal the single-GPU setup's whenever the
// fitted coefficients do; the Gram matrix and the growth norms are summed
// per rank and then over the ranks in rank order (identically in emulation
// and under NCCL), which may move the last bits of those reductions.
//
// Ranks: d.me < 0 runs every rank in this process (one GPU, no kernel waits
// on another rank); d.me >= 0 is one rank per process, the exchanges are
// NCCL grouped send / receive and all-gathers.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "dist.cuh"
#include "sparse.cuh"

namespace airg {

namespace {

__device__ __forceinline__ int owner_s(const int64_t* __restrict__ s, int P, int64_t g) {
  int lo = 0, hi = P;  // largest r with s[r] <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// locality counts (partition_model.cpp:53-64) of local rows base.. against
// the partition s: [r] entries on the row's owner, [P + r] off it
__global__ void k_locality_rows(int n, int64_t base, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const int64_t* __restrict__ s, int P, unsigned long long* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = owner_s(s, P, base + i);
  unsigned long long loc = 0, non = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) (owner_s(s, P, ci[k]) == r ? loc : non)++;
  if (loc) atomicAdd(cnt + r, loc);
  if (non) atomicAdd(cnt + P + r, non);
}

// rows `want` of the ranks' slabs (s: starts, tables of the slabs' arrays)
__global__ void k_fetch_len(int64_t nw, const int32_t* __restrict__ want, const int64_t* __restrict__ s, int P,
                            const int32_t* const* __restrict__ rps, int32_t* __restrict__ len) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nw) return;
  const int64_t g = want[k];
  const int q = owner_s(s, P, g);
  const int64_t row = g - s[q];
  len[k] = rps[q][row + 1] - rps[q][row];
}
__global__ void k_fetch_fill(int64_t nw, const int32_t* __restrict__ want, const int64_t* __restrict__ s, int P,
                             const int32_t* const* __restrict__ rps, const int32_t* const* __restrict__ cis,
                             const double* const* __restrict__ vs, const int32_t* __restrict__ orp,
                             int32_t* __restrict__ oci, double* __restrict__ ov) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nw) return;
  const int64_t g = want[k];
  const int q = owner_s(s, P, g);
  const int64_t row = g - s[q];
  const int32_t* rp = rps[q];
  int o = orp[k];
  for (int t = rp[row]; t < rp[row + 1]; ++t) {
    oci[o] = cis[q][t];
    ov[o++] = vs[q][t];
  }
}

__global__ void k_iota(int64_t n, int64_t base, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = (int32_t)(base + k);
}

// F flags of the own rows and their prefix -> global F / C numbers:
// code = f (F point) or -(c + 1) (C point)
__global__ void k_isf(int64_t n, const double* __restrict__ lab, int32_t* __restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = lab[i] == (double)AIRG_F;
}
__global__ void k_codes(int64_t n, const double* __restrict__ lab, const int32_t* __restrict__ fpos, int64_t flo,
                        int64_t clo, double* __restrict__ code) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (lab[i] == (double)AIRG_F)
    code[i] = (double)(flo + fpos[i]);
  else
    code[i] = -(double)(clo + (i - fpos[i])) - 1.0;
}
// per [own | halo] column: kind (F number or -(C number) - 1), label byte,
// coarse number (C) and global fine index
__global__ void k_colinfo(int64_t nt, const double* __restrict__ code, int64_t lo, int64_t own,
                          const int32_t* __restrict__ halo, int32_t* __restrict__ kind, uint8_t* __restrict__ label,
                          int32_t* __restrict__ cnum, int32_t* __restrict__ gid) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nt) return;
  const int32_t k = (int32_t)code[j];
  kind[j] = k;
  label[j] = k >= 0 ? AIRG_F : AIRG_C;
  cnum[j] = k >= 0 ? -1 : -k - 1;
  gid[j] = j < own ? (int32_t)(lo + j) : halo[j - own];
}

// the blocks of the own rows (extract_blocks, cfsplit.cu) in the local
// layout: ff / fc / cf counts per own F / C row (ordinal within the rank)
__global__ void k_blk_count(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ kind, int64_t flo, int64_t clo, int32_t* __restrict__ ff,
                            int32_t* __restrict__ fc, int32_t* __restrict__ cf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int nF = 0, nC = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) (kind[ci[k]] >= 0 ? nF : nC)++;
  const int32_t ki = kind[i];
  if (ki >= 0) {
    ff[ki - flo] = nF;
    fc[ki - flo] = nC;
  } else {
    cf[(-ki - 1) - clo] = nF;
  }
}
__global__ void k_blk_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, const int32_t* __restrict__ kind,
                           const int32_t* __restrict__ gid, int64_t flo, int64_t clo,
                           const int32_t* __restrict__ ffrp, int32_t* __restrict__ ffci, int32_t* __restrict__ ffgci,
                           double* __restrict__ ffv, double* __restrict__ ffgv, const int32_t* __restrict__ fcrp,
                           int32_t* __restrict__ fcci, double* __restrict__ fcv, const int32_t* __restrict__ cfrp,
                           int32_t* __restrict__ cfci, double* __restrict__ cfv, const int32_t* __restrict__ afrp,
                           int32_t* __restrict__ afci, double* __restrict__ afv, int32_t* __restrict__ f2f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t ki = kind[i];
  if (ki >= 0) {
    const int64_t r = ki - flo;
    f2f[r] = gid[i];
    int of = ffrp[r], oc = fcrp[r], oa = afrp[r];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t j = ci[k], kj = kind[j];
      if (kj >= 0) {
        ffci[of] = kj;
        ffgci[of] = gid[j];
        ffv[of] = v[k];
        ffgv[of++] = v[k];
        afci[oa] = gid[j];
      } else {
        fcci[oc] = -kj - 1;
        fcv[oc++] = v[k];
        afci[oa] = (int32_t)((unsigned)gid[j] | 0x80000000u);
      }
      afv[oa++] = v[k];
    }
  } else {
    int o = cfrp[(-ki - 1) - clo];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t kj = kind[ci[k]];
      if (kj >= 0) {
        cfci[o] = kj;
        cfv[o++] = v[k];
      }
    }
  }
}
__global__ void k_add2(int64_t n, const int32_t* __restrict__ a, const int32_t* __restrict__ b, int32_t* __restrict__ o) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) o[k] = a[k] + b[k];
}

// columns -> a layout: own [lo, lo + own) at base + (g - lo), the sorted
// halo h[p] at p (p < nb) or own + p (p >= nb); not found -> -1. nb = 0 and
// base = 0 give the [own | halo] layout.
__global__ void k_to_layout(int64_t nnz, const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t lo,
                            int64_t own, const int32_t* __restrict__ h, int64_t nh, int64_t nb) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int64_t g = in[k] & 0x7fffffff;
  if (g >= lo && g < lo + own) {
    out[k] = (int32_t)(nb + (g - lo));
    return;
  }
  int64_t a = 0, b = nh;
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (h[m] < g)
      a = m + 1;
    else
      b = m;
  }
  out[k] = (a < nh && h[a] == g) ? (int32_t)(a < nb ? a : own + a) : -1;
}
// layout index -> a value: own rows from `own_val`, halo from `halo_val`
__global__ void k_from_layout(int64_t nnz, int32_t* __restrict__ ci, const int32_t* __restrict__ own_val,
                              int64_t own, const int32_t* __restrict__ halo_val, int64_t nb) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int64_t e = ci[k];
  if (e < nb)
    ci[k] = halo_val[e];
  else if (e < nb + own)
    ci[k] = own_val[e - nb];
  else
    ci[k] = halo_val[e - own];
}

__global__ void k_d2i(int64_t n, const double* __restrict__ in, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = (int32_t)in[k];
}
__global__ void k_i2d(int64_t n, const int32_t* __restrict__ in, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = (double)in[k];
}
__global__ void k_count_ge0(int64_t n, const int32_t* __restrict__ x, unsigned long long* __restrict__ cnt) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  block_add(cnt, (k < n && x[k] >= 0) ? 1ull : 0ull);
}
// fmap[F number] = fine index of every A_ff entry (the halo F points' fine indices)
__global__ void k_scatter_fine(int64_t nnz, const int32_t* __restrict__ fci, const int32_t* __restrict__ gci,
                               int32_t* __restrict__ fmap) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) fmap[fci[k]] = gci[k];
}
__global__ void k_gather_i32(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ src,
                             int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = src[idx[k]];
}

// ---- growth guard reductions: block partials -> one per rank -> rank order
__global__ void k_sub_norm_part(int n, double* __restrict__ v, const double* __restrict__ q,
                                double* __restrict__ part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = q ? v[i] - q[i] : v[i];
    v[i] = x;
    s += x * x;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}
__global__ void k_sum_ordered(const double* __restrict__ part, int np, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += part[i];
    *out = s;
  }
}
__global__ void k_sqrt_to(const double* __restrict__ all, int P, double* __restrict__ g) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < P; ++r) s += all[r];
    *g = sqrt(s);
  }
}
__global__ void k_scale(int n, double* __restrict__ v, const double* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double gg = *g;
  if (i < n && gg != 0.0) v[i] = v[i] / gg;
}

// ---------------------------------------------------------------------------
template <class F>
void each(const DHier& d, F&& f) {
  for (int r = 0; r < d.P; ++r)
    if (d.mine(r)) f(r);
}

void empty_rows(Ctx& c, Csr& m, int64_t ncols) {
  m = Csr();
  m.n = 0;
  m.m = (int32_t)ncols;
  m.nnz = 0;
  m.rp.alloc(c, 1);
  m.rp.zero(c);
}

// k values per rank: v holds P * k entries; under NCCL the rank's own k are
// filled on entry, every rank's on return (emulation: all filled already)
template <class T>
void allgather(Ctx& c, const DHier& d, std::vector<T>& v, int k) {
  if (d.me < 0 || d.P == 1) return;
  static_assert(sizeof(T) == 8, "8-byte values");
  DBuf<T> mine(c, (size_t)k), all(c, (size_t)k * d.P);
  to_device(c, mine.p, v.data() + (size_t)d.me * k, (size_t)k);
  NCCL_CHECK(ncclAllGather(mine.p, all.p, (size_t)k, ncclInt64, d.comm, c.stream));
  to_host(c, v.data(), all.p, (size_t)k * d.P);
}

// per-rank device scalars slot[r] (emulation: all P in one buffer written
// by the ranks; NCCL: this rank's at slot[me]) -> all P on every rank
void gather_scalars(Ctx& c, const DHier& d, double* slot) {
  if (d.me < 0 || d.P == 1) return;
  NCCL_CHECK(ncclAllGather(slot + d.me, slot, 1, ncclDouble, d.comm, c.stream));
}

// Rows want[r] (sorted global rows, nwant[r] of them) of the row-partitioned
// matrix M (M[q]: rows part.lo(q).. of rank q, ranks of this process) into
// out[r], columns unchanged (the halo-row gather of the setup).
void fetch_rows(Ctx& c, const DHier& d, const Part& part, std::vector<Csr>& M, int64_t ncols,
                std::vector<DBuf<int32_t>>& want, const std::vector<int64_t>& nwant, std::vector<Csr>& out) {
  const int P = d.P;
  out.resize(P);
  DBuf<int64_t> ds(c, (size_t)P + 1);
  to_device(c, ds.p, part.s.data(), (size_t)P + 1);
  auto alloc_out = [&](Csr& o, int64_t nw) {
    o = Csr();
    o.n = (int32_t)nw;
    o.m = (int32_t)ncols;
    o.rp.alloc(c, (size_t)nw + 1);
  };
  if (d.me < 0 || P == 1) {
    std::vector<const int32_t*> hrp(P, nullptr), hci(P, nullptr);
    std::vector<const double*> hv(P, nullptr);
    for (int q = 0; q < P; ++q)
      if (d.mine(q)) {
        hrp[q] = M[q].rp.p;
        hci[q] = M[q].ci.p;
        hv[q] = M[q].v.p;
      }
    DBuf<const int32_t*> rps(c, (size_t)P), cis(c, (size_t)P);
    DBuf<const double*> vs(c, (size_t)P);
    to_device(c, rps.p, hrp.data(), (size_t)P);
    to_device(c, cis.p, hci.data(), (size_t)P);
    to_device(c, vs.p, hv.data(), (size_t)P);
    each(d, [&](int r) {
      const int64_t nw = nwant[r];
      Csr& o = out[r];
      alloc_out(o, nw);
      DBuf<int32_t> len(c, (size_t)std::max<int64_t>(1, nw));
      if (nw) LAUNCH(c, k_fetch_len, blocks_for(nw, 256), 256, 0, nw, want[r].p, ds.p, P, rps.p, len.p);
      o.nnz = nw ? exclusive_scan(c, len.p, o.rp.p, nw) : 0;
      if (!nw) o.rp.zero(c);
      o.ci.alloc(c, (size_t)o.nnz);
      o.v.alloc(c, (size_t)o.nnz);
      if (nw)
        LAUNCH(c, k_fetch_fill, blocks_for(nw, 128), 128, 0, nw, want[r].p, ds.p, P, rps.p, cis.p, vs.p, o.rp.p,
               o.ci.p, o.v.p);
    });
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return;
  }
  // one rank per process: requests to the owners, lengths back, rows back
  const int me = d.me;
  const int64_t nw = nwant[me];
  std::vector<int32_t> wh((size_t)nw);
  to_host(c, wh.data(), want[me].p, (size_t)nw);
  std::vector<int64_t> wcnt(P, 0), woff(P + 1, 0);
  for (int32_t g : wh) wcnt[part.owner(g)]++;
  for (int q = 0; q < P; ++q) woff[q + 1] = woff[q] + wcnt[q];
  std::vector<int64_t> C((size_t)P * P, 0);
  for (int q = 0; q < P; ++q) C[(size_t)me * P + q] = wcnt[q];
  allgather(c, d, C, P);
  std::vector<int64_t> ask(P, 0), aoff(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    ask[q] = q == me ? 0 : C[(size_t)q * P + me];
    aoff[q + 1] = aoff[q] + ask[q];
  }
  const int64_t na = aoff[P];
  DBuf<int32_t> req(c, (size_t)std::max<int64_t>(1, na));
  NCCL_CHECK(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    if (wcnt[q]) NCCL_CHECK(ncclSend(want[me].p + woff[q], (size_t)wcnt[q], ncclInt32, q, d.comm, c.stream));
    if (ask[q]) NCCL_CHECK(ncclRecv(req.p + aoff[q], (size_t)ask[q], ncclInt32, q, d.comm, c.stream));
  }
  NCCL_CHECK(ncclGroupEnd());
  // my slab as a one-rank table
  const int64_t my_s[2] = {part.lo(me), part.lo(me) + part.cnt(me)};
  DBuf<int64_t> ms(c, 2);
  to_device(c, ms.p, my_s, 2);
  const int32_t* hrp = M[me].rp.p;
  const int32_t* hci = M[me].ci.p;
  const double* hv = M[me].v.p;
  DBuf<const int32_t*> rps(c, 1), cis(c, 1);
  DBuf<const double*> vs(c, 1);
  to_device(c, rps.p, &hrp, 1);
  to_device(c, cis.p, &hci, 1);
  to_device(c, vs.p, &hv, 1);
  DBuf<int32_t> alen(c, (size_t)std::max<int64_t>(1, na)), arp(c, (size_t)na + 1);
  if (na) LAUNCH(c, k_fetch_len, blocks_for(na, 256), 256, 0, na, req.p, ms.p, 1, rps.p, alen.p);
  const int64_t anz = na ? exclusive_scan(c, alen.p, arp.p, na) : 0;
  Csr& o = out[me];
  alloc_out(o, nw);
  DBuf<int32_t> len(c, (size_t)std::max<int64_t>(1, nw));
  if (wcnt[me])
    LAUNCH(c, k_fetch_len, blocks_for(wcnt[me], 256), 256, 0, wcnt[me], want[me].p + woff[me], ms.p, 1, rps.p,
           len.p + woff[me]);
  NCCL_CHECK(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    if (ask[q]) NCCL_CHECK(ncclSend(alen.p + aoff[q], (size_t)ask[q], ncclInt32, q, d.comm, c.stream));
    if (wcnt[q]) NCCL_CHECK(ncclRecv(len.p + woff[q], (size_t)wcnt[q], ncclInt32, q, d.comm, c.stream));
  }
  NCCL_CHECK(ncclGroupEnd());
  o.nnz = nw ? exclusive_scan(c, len.p, o.rp.p, nw) : 0;
  if (!nw) o.rp.zero(c);
  o.ci.alloc(c, (size_t)o.nnz);
  o.v.alloc(c, (size_t)o.nnz);
  std::vector<int32_t> orp_h((size_t)nw + 1), arp_h((size_t)na + 1, 0);
  to_host(c, orp_h.data(), o.rp.p, (size_t)nw + 1);
  if (na) to_host(c, arp_h.data(), arp.p, (size_t)na + 1);
  DBuf<int32_t> pci(c, (size_t)std::max<int64_t>(1, anz));
  DBuf<double> pv(c, (size_t)std::max<int64_t>(1, anz));
  if (na) LAUNCH(c, k_fetch_fill, blocks_for(na, 128), 128, 0, na, req.p, ms.p, 1, rps.p, cis.p, vs.p, arp.p, pci.p, pv.p);
  if (wcnt[me])
    LAUNCH(c, k_fetch_fill, blocks_for(wcnt[me], 128), 128, 0, wcnt[me], want[me].p + woff[me], ms.p, 1, rps.p,
           cis.p, vs.p, o.rp.p + woff[me], o.ci.p, o.v.p);
  NCCL_CHECK(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const int64_t s0 = arp_h[aoff[q]], s1 = arp_h[aoff[q + 1]];
    if (s1 > s0) {
      NCCL_CHECK(ncclSend(pci.p + s0, (size_t)(s1 - s0), ncclInt32, q, d.comm, c.stream));
      NCCL_CHECK(ncclSend(pv.p + s0, (size_t)(s1 - s0), ncclDouble, q, d.comm, c.stream));
    }
    const int64_t r0 = orp_h[woff[q]], r1 = orp_h[woff[q + 1]];
    if (r1 > r0) {
      NCCL_CHECK(ncclRecv(o.ci.p + r0, (size_t)(r1 - r0), ncclInt32, q, d.comm, c.stream));
      NCCL_CHECK(ncclRecv(o.v.p + r0, (size_t)(r1 - r0), ncclDouble, q, d.comm, c.stream));
    }
  }
  NCCL_CHECK(ncclGroupEnd());
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// Rows want[0..nw) (global indices inside [lo, lo + m.n)) of m, in that
// order, columns unchanged.
void select_rows(Ctx& c, const Csr& m, int64_t lo, const int32_t* want, int64_t nw, Csr& out) {
  out = Csr();
  out.n = (int32_t)nw;
  out.m = m.m;
  out.rp.alloc(c, (size_t)nw + 1);
  const int64_t s[2] = {lo, lo + m.n};
  DBuf<int64_t> ms(c, 2);
  to_device(c, ms.p, s, 2);
  const int32_t* hrp = m.rp.p;
  const int32_t* hci = m.ci.p;
  const double* hv = m.v.p;
  DBuf<const int32_t*> rps(c, 1), cis(c, 1);
  DBuf<const double*> vs(c, 1);
  to_device(c, rps.p, &hrp, 1);
  to_device(c, cis.p, &hci, 1);
  to_device(c, vs.p, &hv, 1);
  DBuf<int32_t> len(c, (size_t)std::max<int64_t>(1, nw));
  if (nw) LAUNCH(c, k_fetch_len, blocks_for(nw, 256), 256, 0, nw, want, ms.p, 1, rps.p, len.p);
  out.nnz = nw ? exclusive_scan(c, len.p, out.rp.p, nw) : 0;
  if (!nw) out.rp.zero(c);
  out.ci.alloc(c, (size_t)out.nnz);
  out.v.alloc(c, (size_t)out.nnz);
  if (nw)
    LAUNCH(c, k_fetch_fill, blocks_for(nw, 128), 128, 0, nw, want, ms.p, 1, rps.p, cis.p, vs.p, out.rp.p, out.ci.p,
           out.v.p);
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// Move the rows of M (partition from) to the partition to.
void migrate(Ctx& c, const DHier& d, const Part& from, const Part& to, std::vector<Csr>& M, int64_t ncols) {
  if (from.s == to.s) return;
  const int P = d.P;
  std::vector<DBuf<int32_t>> want(P);
  std::vector<int64_t> nw(P, 0);
  each(d, [&](int r) {
    nw[r] = to.cnt(r);
    want[r].alloc(c, (size_t)std::max<int64_t>(1, nw[r]));
    if (nw[r]) LAUNCH(c, k_iota, blocks_for(nw[r], 256), 256, 0, nw[r], to.lo(r), want[r].p);
  });
  std::vector<Csr> out;
  fetch_rows(c, d, from, M, ncols, want, nw, out);
  each(d, [&](int r) { M[r] = std::move(out[r]); });
}

// The ranks' row blocks concatenated in the given order (columns unchanged)
void concat_rows(Ctx& c, const std::vector<const Csr*>& parts, const std::vector<std::pair<int64_t, int64_t>>& rng,
                 int64_t ncols, Csr& out) {
  int64_t n = 0;
  std::vector<int32_t> rbase, rend;
  for (size_t k = 0; k < parts.size(); ++k) n += rng[k].second - rng[k].first;
  out = Csr();
  out.n = (int32_t)n;
  out.m = (int32_t)ncols;
  out.rp.alloc(c, (size_t)n + 1);
  // entry ranges of each piece
  int64_t nnz = 0;
  std::vector<int64_t> e0(parts.size()), e1(parts.size());
  for (size_t k = 0; k < parts.size(); ++k) {
    const auto [a, b] = rng[k];
    int32_t x[2] = {0, 0};
    if (b > a) {
      to_host(c, &x[0], parts[k]->rp.p + a, 1);
      to_host(c, &x[1], parts[k]->rp.p + b, 1);
    }
    e0[k] = x[0];
    e1[k] = x[1];
    nnz += x[1] - x[0];
  }
  out.nnz = nnz;
  out.ci.alloc(c, (size_t)nnz);
  out.v.alloc(c, (size_t)nnz);
  int64_t row = 0, ent = 0;
  std::vector<int32_t> rp_h((size_t)n + 1);
  for (size_t k = 0; k < parts.size(); ++k) {
    const auto [a, b] = rng[k];
    if (b > a) {
      std::vector<int32_t> prp((size_t)(b - a) + 1);
      to_host(c, prp.data(), parts[k]->rp.p + a, prp.size());
      for (int64_t i = 0; i <= b - a; ++i) rp_h[row + i] = (int32_t)(ent + prp[i] - e0[k]);
      const int64_t cnt = e1[k] - e0[k];
      if (cnt) {
        CUDA_CHECK(cudaMemcpyAsync(out.ci.p + ent, parts[k]->ci.p + e0[k], sizeof(int32_t) * cnt,
                                   cudaMemcpyDeviceToDevice, c.stream));
        CUDA_CHECK(cudaMemcpyAsync(out.v.p + ent, parts[k]->v.p + e0[k], sizeof(double) * cnt,
                                   cudaMemcpyDeviceToDevice, c.stream));
      }
      row += b - a;
      ent += cnt;
    }
  }
  rp_h[n] = (int32_t)ent;
  to_device(c, out.rp.p, rp_h.data(), rp_h.size());
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// halo plan of V for rank r from the columns of the given local matrices
// (global columns; own range = V.part's)
void plan_rank(Ctx& c, DVec& V, int r, std::initializer_list<const Csr*> ms) {
  Marks mk;
  mk.init(c, V.N);
  const int64_t lo = V.part.lo(r), hi = lo + V.part.cnt(r);
  for (const Csr* m : ms) mk.cols(c, *m, lo, hi);
  set_halo(c, V, r, mk);
}

void to_layout(Ctx& c, Csr& m, const DVec& V, int r, int64_t nb) {
  const DVec::Rank& R = V.rk[r];
  if (m.nnz)
    LAUNCH(c, k_to_layout, blocks_for(m.nnz, 256), 256, 0, m.nnz, m.ci.p, m.ci.p, R.lo, R.own, R.halo.p, R.nhalo, nb);
  m.m = (int32_t)(R.own + R.nhalo);
}

// Distributed locality of the rows held (partition `held`, rows M) against
// the candidate partition p: the reference ratio and local share.
double dist_locality(Ctx& c, const DHier& d, const Part& held, std::vector<Csr>& M, const Part& p, double* share) {
  const int P = d.P;
  DBuf<int64_t> ds(c, (size_t)P + 1);
  to_device(c, ds.p, p.s.data(), (size_t)P + 1);
  std::vector<int64_t> cnt((size_t)P * 2 * P, 0);
  each(d, [&](int r) {
    DBuf<unsigned long long> k(c, (size_t)2 * P);
    k.zero(c);
    if (M[r].n)
      LAUNCH(c, k_locality_rows, blocks_for(M[r].n, 256), 256, 0, M[r].n, held.lo(r), M[r].rp.p, M[r].ci.p, ds.p, P,
             k.p);
    std::vector<unsigned long long> h((size_t)2 * P);
    to_host(c, h.data(), k.p, h.size());
    for (int x = 0; x < 2 * P; ++x) cnt[(size_t)r * 2 * P + x] = (int64_t)h[x];
  });
  allgather(c, d, cnt, 2 * P);
  std::vector<unsigned long long> tot((size_t)2 * P, 0);
  for (int r = 0; r < P; ++r)
    for (int x = 0; x < 2 * P; ++x) tot[x] += (unsigned long long)cnt[(size_t)r * 2 * P + x];
  // locality() (dist.cu) on the summed counts
  if (share) *share = 1.0;
  int64_t n = p.s[P];
  if (n == 0) return INFINITY;
  double sum = 0.0;
  int contributing = 0;
  unsigned long long loc = 0, all = 0;
  for (int r = 0; r < P; ++r) {
    loc += tot[r];
    all += tot[r] + tot[P + r];
    if (tot[P + r] == 0) continue;
    sum += (double)tot[r] / (double)tot[P + r];
    ++contributing;
  }
  if (share && all) *share = (double)loc / (double)all;
  return contributing ? sum / contributing : INFINITY;
}

int64_t sum_over_ranks(Ctx& c, const DHier& d, std::vector<int64_t> v) {
  allgather(c, d, v, 1);
  int64_t s = 0;
  for (int64_t x : v) s += x;
  return s;
}

// ---- the distributed polynomial inverse of A_ff (F partition fp) ----------
struct FfRank {
  Csr aff;       // own F rows, global F columns
  Csr affc;      // the same, [own | halo] layout of VF
  Csr ext;       // [halo below | own | halo above] rows, columns in that (sorted) layout
  int64_t nb = 0;
  std::vector<int64_t> halo_host;
};

struct DistInverse {
  std::vector<double> coeffs;
  int64_t eff = 0, attempts = 1;
  double growth = 0.0;
  std::vector<Csr> q;  // own F rows, global F columns
};

// rows of the assembly for every rank with the given coefficients
void assemble_owned(Ctx& c, const DHier& d, std::vector<FfRank>& fr, const DVec& VF, const std::vector<double>& coeffs,
                    int64_t eff, std::vector<Csr>& q) {
  q.resize(d.P);
  each(d, [&](int r) {
    const DVec::Rank& R = VF.rk[r];
    Csr out;
    poly_assemble_rows(c, fr[r].ext, (int)fr[r].nb, (int)R.own, coeffs.data(), (int64_t)coeffs.size(), eff, out);
    // layout -> global F numbers: own rows lo.., halo from the sorted list
    DBuf<int32_t> ownv(c, (size_t)std::max<int64_t>(1, R.own));
    if (R.own) LAUNCH(c, k_iota, blocks_for(R.own, 256), 256, 0, R.own, R.lo, ownv.p);
    if (out.nnz)
      LAUNCH(c, k_from_layout, blocks_for(out.nnz, 256), 256, 0, out.nnz, out.ci.p, ownv.p, R.own, R.halo.p, fr[r].nb);
    out.m = (int32_t)VF.N;
    q[r] = std::move(out);
  });
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// y = M x over the ranks: x own -> V [own | halo] -> y own
void dist_spmv(Ctx& c, DHier& d, DVec& V, std::vector<Csr>& Mc, std::vector<DBuf<double>>& x,
               std::vector<DBuf<double>>& y) {
  each(d, [&](int r) {
    DVec::Rank& R = V.rk[r];
    if (R.own) CUDA_CHECK(cudaMemcpyAsync(R.buf.p, x[r].p, sizeof(double) * R.own, cudaMemcpyDeviceToDevice, c.stream));
  });
  exchange(c, d, V);
  each(d, [&](int r) {
    if (Mc[r].n) spmv(c, Mc[r], V.rk[r].buf.p, y[r].p);
  });
}

double dist_growth(Ctx& c, DHier& d, DVec& VF, std::vector<Csr>& affc, std::vector<Csr>& qc) {
  const int P = d.P;
  constexpr int kIters = 30, kTail = 15;
  const int64_t N = VF.N;
  if (N == 0) return 0.0;
  std::vector<DBuf<double>> v(P), av(P), qav(P), part(P);
  DBuf<double> all(c, (size_t)P), g(c, kIters + 1);
  all.zero(c);
  const int threads = 256;
  const uint64_t probe_seed = mix_host(0xA3B1C5D7ull, (uint64_t)N);
  std::vector<int> blocks(P, 1);
  each(d, [&](int r) {
    const int64_t n = VF.rk[r].own;
    v[r].alloc(c, (size_t)std::max<int64_t>(1, n));
    av[r].alloc(c, (size_t)std::max<int64_t>(1, n));
    qav[r].alloc(c, (size_t)std::max<int64_t>(1, n));
    blocks[r] = (int)std::max<int64_t>(1, std::min<int64_t>(kReduceBlocks, blocks_for(n, threads)));
    part[r].alloc(c, (size_t)blocks[r]);
    poly_basis_fill(c, n, VF.rk[r].lo, probe_seed, v[r].p, nullptr);
  });
  auto norm_scale = [&](int k, bool sub) {
    each(d, [&](int r) {
      const int n = (int)VF.rk[r].own;
      LAUNCH(c, k_sub_norm_part, blocks[r], threads, 0, n, v[r].p, sub ? (const double*)qav[r].p : nullptr, part[r].p);
      LAUNCH(c, k_sum_ordered, 1, 32, 0, part[r].p, blocks[r], all.p + r);
    });
    gather_scalars(c, d, all.p);
    LAUNCH(c, k_sqrt_to, 1, 32, 0, all.p, P, g.p + k);
    each(d, [&](int r) {
      const int n = (int)VF.rk[r].own;
      if (n) LAUNCH(c, k_scale, blocks_for(n, 256), 256, 0, n, v[r].p, g.p + k);
    });
  };
  norm_scale(kIters, false);
  for (int k = 0; k < kIters; ++k) {
    dist_spmv(c, d, VF, affc, v, av);
    dist_spmv(c, d, VF, qc, av, qav);
    norm_scale(k, true);
  }
  double hg[kIters + 1];
  to_host(c, hg, g.p, kIters + 1);
  double log_growth = 0.0;
  int tail = 0;
  for (int k = 0; k < kIters; ++k) {
    if (hg[k] == 0.0) return 0.0;
    if (k >= kTail) {
      log_growth += std::log(hg[k]);
      ++tail;
    }
  }
  return std::exp(log_growth / tail);
}

PolyFit dist_fit(Ctx& c, DHier& d, DVec& VF, std::vector<Csr>& affc, int64_t m, uint64_t seed) {
  const int P = d.P;
  const int64_t N = VF.N;
  if (N == 0) throw InvalidArgument("compute_coefficients: empty matrix");
  const int nc = (int)(m + 1);
  const uint64_t rhs_seed = mix_host(seed, 0x504f4c59ull);
  std::vector<DBuf<double>> kh(P), kl(P), eh(P), el(P);
  each(d, [&](int r) {
    const DVec::Rank& R = VF.rk[r];
    const int64_t n = R.own;
    kh[r].alloc(c, (size_t)std::max<int64_t>(1, n * nc));
    kl[r].alloc(c, (size_t)std::max<int64_t>(1, n * nc));
    eh[r].alloc(c, (size_t)std::max<int64_t>(1, R.own + R.nhalo));
    el[r].alloc(c, (size_t)std::max<int64_t>(1, R.own + R.nhalo));
    poly_basis_fill(c, n, R.lo, rhs_seed, kh[r].p, kl[r].p);
  });
  auto halo_of = [&](std::vector<DBuf<double>>& src, int k, std::vector<DBuf<double>>& dst) {
    each(d, [&](int r) {
      DVec::Rank& R = VF.rk[r];
      if (R.own)
        CUDA_CHECK(cudaMemcpyAsync(R.buf.p, src[r].p + (int64_t)k * R.own, sizeof(double) * R.own,
                                   cudaMemcpyDeviceToDevice, c.stream));
    });
    exchange(c, d, VF);
    each(d, [&](int r) {
      DVec::Rank& R = VF.rk[r];
      const int64_t t = R.own + R.nhalo;
      if (t) CUDA_CHECK(cudaMemcpyAsync(dst[r].p, R.buf.p, sizeof(double) * t, cudaMemcpyDeviceToDevice, c.stream));
    });
  };
  for (int k = 1; k <= m; ++k) {
    halo_of(kh, k - 1, eh);
    halo_of(kl, k - 1, el);
    each(d, [&](int r) {
      const int64_t n = VF.rk[r].own;
      poly_dd_spmv(c, affc[r], eh[r].p, el[r].p, kh[r].p + k * n, kl[r].p + k * n);
    });
  }
  // Gram per rank, then over the ranks in rank order (every rank the same)
  std::vector<double> parts((size_t)P * nc * nc * 2, 0.0);
  each(d, [&](int r) {
    std::vector<dd> G;
    poly_gram(c, VF.rk[r].own, nc, kh[r].p, kl[r].p, G);
    for (size_t i = 0; i < G.size(); ++i) {
      parts[((size_t)r * nc * nc + i) * 2] = G[i].hi;
      parts[((size_t)r * nc * nc + i) * 2 + 1] = G[i].lo;
    }
  });
  allgather(c, d, parts, nc * nc * 2);
  std::vector<dd> G((size_t)nc * nc, dd{0.0, 0.0});
  for (int r = 0; r < P; ++r)
    for (size_t i = 0; i < G.size(); ++i)
      G[i] = dd_add(G[i], dd{parts[((size_t)r * nc * nc + i) * 2], parts[((size_t)r * nc * nc + i) * 2 + 1]});
  return poly_fit_gram(G, nc, m, N);
}

// make_checked_inverse (air.cpp:106-129) over the ranks
DistInverse dist_checked_inverse(Ctx& c, DHier& d, DVec& VF, std::vector<FfRank>& fr, std::vector<Csr>& affc,
                                 int64_t order, uint64_t seed, const std::vector<double>* fixed, int64_t fixed_eff) {
  const int P = d.P;
  DistInverse best;
  if (fixed) {
    best.coeffs = *fixed;
    best.eff = fixed_eff;
    assemble_owned(c, d, fr, VF, best.coeffs, best.eff, best.q);
    return best;
  }
  double best_growth = INFINITY;
  for (int64_t attempt = 0; attempt < 6; ++attempt) {
    const uint64_t s = attempt == 0 ? seed : mix_host(seed, 0x52455452ull + (uint64_t)attempt);
    PolyFit fit = dist_fit(c, d, VF, affc, order + 1, s);
    std::vector<Csr> q;
    assemble_owned(c, d, fr, VF, fit.coeffs, fit.effective_order, q);
    std::vector<Csr> qc(P);
    each(d, [&](int r) {
      csr_copy(c, q[r], qc[r]);
      to_layout(c, qc[r], VF, r, 0);
    });
    const double growth = dist_growth(c, d, VF, affc, qc);
    if (growth < best_growth) {
      best.coeffs = fit.coeffs;
      best.eff = fit.effective_order;
      best.q = std::move(q);
      best.growth = growth;
      best.attempts = attempt + 1;
      best_growth = growth;
    }
    if (best_growth <= 0.5) break;
  }
  return best;
}

}  // namespace

void dist_setup_owned(Ctx& c, std::vector<Csr>& a_rows, const std::vector<int64_t>& starts,
                      const airg_setup_config& cfg, const Injection* inj, int P, int me, ncclComm_t comm,
                      double threshold, DHier& d) {
  NvtxRange nvtx__("airg dist setup (owned)");
  if (P < 1) throw InvalidArgument("dist: need at least one rank");
  if (me >= P) throw InvalidArgument("dist: rank out of range");
  if (me >= 0 && P > 1 && !comm) throw InvalidArgument("dist: a communicator is needed per rank");
  if ((int)starts.size() != P + 1 || starts[0] != 0) throw InvalidArgument("dist: slab starts must cover the matrix");
  if (cfg.poly_order < 1 || cfg.coarse_poly_order < 1) throw InvalidArgument("setup: polynomial orders must be >= 1");
  if (cfg.sparsity_order != 1)
    throw InvalidArgument("owned distributed setup: sparsity_order 1 only (the A_ff halo is distance 1)");
  if (cfg.cf != 0 || cfg.weight_mode != 0)
    throw InvalidArgument("owned distributed setup: PMISR with |S| + |S^T| weights only");
  if (cfg.ddc_enabled && !(cfg.ddc_fraction > 0.0 && cfg.ddc_fraction <= 1.0))
    throw InvalidArgument("ddc: fraction must be in (0, 1]");
  if (cfg.drop_coarse < 0.0 || cfg.drop_restrict < 0.0) throw InvalidArgument("setup: drop tolerances must be >= 0");
  if (cfg.strength_alpha < 0.0 || cfg.strength_alpha > 1.0)
    throw InvalidArgument("setup: strength_alpha must lie in [0, 1]");
  if (cfg.prolongation != 0) throw InvalidArgument("setup: the GPU path implements one-point prolongation only");
  if (cfg.poly_order + 1 > 32 || cfg.coarse_poly_order + 1 > 32)
    throw InvalidArgument("setup: polynomial order above 31 not supported");
  const auto t_start = std::chrono::steady_clock::now();
  cudaEvent_t ev0, ev1;
  CUDA_CHECK(cudaEventCreate(&ev0));
  CUDA_CHECK(cudaEventCreate(&ev1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } evg{ev0, ev1};
  d.cf_ms = 0.0;
  const int64_t N0 = starts[P];
  d.P = P;
  d.me = me;
  d.comm = comm;
  d.threshold = threshold;
  d.owned = true;
  d.top_n = N0;
  d.lv.clear();
  d.summary.clear();
  const int64_t min_rows = [] {
    const char* e = getenv("AIRG_DIST_MIN_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();

  DistPieces pc;
  pc.all_ranks = false;
  std::vector<Csr> cur(P);
  Part held;  // partition of cur's rows
  held.s = starts;
  int64_t n_cur = N0;
  each(d, [&](int r) {
    if (a_rows[r].n != held.cnt(r)) throw InvalidArgument("dist: local rows do not match the slab starts");
    if (a_rows[r].m != N0) throw InvalidArgument("dist: local rows must carry global columns");
    with_full_diagonal(c, a_rows[r], cur[r], (int)held.lo(r), true);  // air.cpp:307
  });
  std::vector<Csr> top(P);
  each(d, [&](int r) { csr_copy(c, cur[r], top[r]); });
  // R rows of the previous level, in their coarse-point (induced) partition,
  // moved once the next partition is known
  std::vector<Csr> pending_r;
  Part pending_part;
  int active = P;
  constexpr double kCoarseAccept = 0.5;
  CheckedInverse coarse;
  bool coarse_valid = false;

  // gather the current operator on rank 0 and fit the coarse polynomial
  // there (rank 0's results broadcast: every rank takes the same branch)
  auto coarse_try = [&](int64_t built) {
    const Part g0 = gathered(n_cur, P);
    std::vector<Csr> tmp(P);
    each(d, [&](int r) { csr_copy(c, cur[r], tmp[r]); });
    migrate(c, d, held, g0, tmp, n_cur);
    double info[40] = {};
    CheckedInverse ci;
    if (d.mine(0)) {
      ci = inj ? fixed_inverse(c, tmp[0], inj->coarse_coeffs, inj->coarse_eff, cfg.sparsity_order)
               : checked_inverse(c, tmp[0], cfg.coarse_poly_order, cfg.sparsity_order,
                                 mix_host(cfg.seed, 0xC0A12534ull + (uint64_t)built));
      info[0] = ci.growth;
      info[1] = (double)ci.attempts;
      info[2] = (double)ci.eff;
      info[3] = (double)ci.q.nnz;
      info[4] = (double)ci.coeffs.size();
      for (size_t k = 0; k < ci.coeffs.size() && k < 32; ++k) info[5 + k] = ci.coeffs[k];
    }
    if (me >= 0 && P > 1) {
      DBuf<double> b(c, 40);
      to_device(c, b.p, info, 40);
      NCCL_CHECK(ncclBroadcast(b.p, b.p, 40, ncclDouble, 0, comm, c.stream));
      to_host(c, info, b.p, 40);
    }
    if (!d.mine(0)) {
      ci.growth = info[0];
      ci.attempts = (int64_t)info[1];
      ci.eff = (int64_t)info[2];
      ci.coeffs.assign(info + 5, info + 5 + (int64_t)info[4]);
      empty_rows(c, ci.q, n_cur);
    }
    return std::make_pair(std::move(ci), (int64_t)info[3]);
  };
  int64_t coarse_inv_nnz = 0;

  for (;;) {
    const int64_t built = (int64_t)d.lv.size();
    const bool forced = n_cur <= cfg.poly_order + 1 || (cfg.max_levels > 0 && built + 1 >= cfg.max_levels);
    if (inj) {
      if (built >= inj->n_levels) break;
    } else if (forced || n_cur <= cfg.coarse_size_target) {  // air.cpp:309-320
      auto [ci, qnnz] = coarse_try(built);
      if (forced || ci.growth <= kCoarseAccept) {
        coarse = std::move(ci);
        coarse_valid = true;
        coarse_inv_nnz = qnnz;
        break;
      }
    }
    // ---- the level's partition: balanced over the active ranks, then the
    // replay halving rule (dist_create, partition_model.cpp:77-112)
    DLevel D;
    {
      const bool fixed = built == 0;
      Part p = fixed ? Part{starts} : balanced(n_cur, active, P);
      D.ratio_before = dist_locality(c, d, held, cur, p, &D.share_before);
      D.ratio_after = D.ratio_before;
      D.share_after = D.share_before;
      if (!fixed && D.ratio_before < threshold && active > 1) {
        const int na = (active + 1) / 2;
        p = merged(p, active, na);
        active = na;
        D.triggered = true;
        D.ratio_after = dist_locality(c, d, held, cur, p, &D.share_after);
      }
      while (!fixed && min_rows > 0 && active > 1 && n_cur < min_rows * (int64_t)active) {
        const int na = (active + 1) / 2;
        p = merged(p, active, na);
        active = na;
        D.triggered = true;
        D.ratio_after = dist_locality(c, d, held, cur, p, &D.share_after);
      }
      D.active = active;
      D.fine = p;
      migrate(c, d, held, p, cur, n_cur);
      held = p;
    }
    const uint64_t level_seed = mix_host(cfg.seed, (uint64_t)built);  // air.cpp:324-325
    DHier::Summary S;
    S.n = n_cur;
    {
      std::vector<int64_t> nz(P, 0);
      each(d, [&](int r) { nz[r] = cur[r].nnz; });
      S.nnz = sum_over_ranks(c, d, nz);
    }

    // ---- CF split on the slabs (dist.cu), labels over [own | halo]
    DVec V;
    V.part = held;
    V.N = n_cur;
    V.rk.resize(P);
    std::vector<Csr> loc(P);
    each(d, [&](int r) { plan_rank(c, V, r, {&cur[r]}); });
    finalize(c, V, d, false);
    each(d, [&](int r) {
      csr_copy(c, cur[r], loc[r]);
      remap(c, loc[r], V, r);
    });
    CfReport rep;
    std::vector<DBuf<double>> labs;
    CUDA_CHECK(cudaEventRecord(ev0, c.stream));
    cf_split_slabs(c, d, V, loc, cfg.strength_alpha, level_seed, cfg.ddc_enabled != 0, cfg.ddc_fraction,
                   cfg.ddc_bins, labs, rep);
    CUDA_CHECK(cudaEventRecord(ev1, c.stream));
    CUDA_CHECK(cudaEventSynchronize(ev1));
    {
      float ms = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&ms, ev0, ev1));
      d.cf_ms += ms;
    }
    S.n_f_pre = rep.n_f_pre;
    S.n_converted = rep.n_converted;
    S.alpha_diag = rep.alpha_diag;
    S.max_theta_pre = rep.max_theta;

    // ---- global F / C numbers: counts over the ranks, prefix, exchange
    std::vector<int64_t> nfr((size_t)P, 0);
    std::vector<DBuf<int32_t>> fpos(P);
    each(d, [&](int r) {
      const int64_t n = V.rk[r].own;
      DBuf<int32_t> isf(c, (size_t)std::max<int64_t>(1, n));
      fpos[r].alloc(c, (size_t)n + 1);
      if (n) LAUNCH(c, k_isf, blocks_for(n, 256), 256, 0, n, labs[r].p, isf.p);
      nfr[r] = n ? exclusive_scan(c, isf.p, fpos[r].p, n) : 0;
      if (!n) fpos[r].zero(c);
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });
    allgather(c, d, nfr, 1);
    std::vector<int64_t> flo(P + 1, 0), clo(P + 1, 0);
    for (int r = 0; r < P; ++r) {
      flo[r + 1] = flo[r] + nfr[r];
      clo[r + 1] = clo[r] + (held.cnt(r) - nfr[r]);
    }
    const int64_t nf = flo[P], nc = clo[P];
    S.nf = nf;
    S.nc = nc;
    // stall guards (air.cpp:362-376)
    if (nf == 0)
      throw RuntimeError("setup: coarsening stall, no F points selected on level " + std::to_string(built));
    if (nc == 0) break;  // all F: this operator is the coarse grid (air.cpp:538-543)
    if ((double)nc > 0.99 * (double)n_cur)
      throw RuntimeError("setup: coarsening stall, level " + std::to_string(built) + " coarsened by less than 1% (" +
                         std::to_string(n_cur) + " -> " + std::to_string(nc) + ")");
    if (built > 0) {  // a level is built: the previous level's R rows to its partition
      migrate(c, d, pending_part, held, pending_r, pc.n.back());
      each(d, [&](int r) { pc.lv.back()[r].R = std::move(pending_r[r]); });
    }
    each(d, [&](int r) {
      DVec::Rank& R = V.rk[r];
      if (R.own) LAUNCH(c, k_codes, blocks_for(R.own, 256), 256, 0, R.own, labs[r].p, fpos[r].p, flo[r], clo[r], R.buf.p);
    });
    exchange(c, d, V);
    struct ColInfo {
      DBuf<int32_t> kind, cnum, gid;
      DBuf<uint8_t> label;
    };
    std::vector<ColInfo> ci(P);
    each(d, [&](int r) {
      DVec::Rank& R = V.rk[r];
      const int64_t t = std::max<int64_t>(1, R.own + R.nhalo);
      ci[r].kind.alloc(c, (size_t)t);
      ci[r].cnum.alloc(c, (size_t)t);
      ci[r].gid.alloc(c, (size_t)t);
      ci[r].label.alloc(c, (size_t)t);
      if (R.own + R.nhalo)
        LAUNCH(c, k_colinfo, blocks_for(R.own + R.nhalo, 256), 256, 0, R.own + R.nhalo, R.buf.p, R.lo, R.own,
               R.halo.p, ci[r].kind.p, ci[r].label.p, ci[r].cnum.p, ci[r].gid.p);
    });

    // ---- blocks of the own rows
    Part fpart, cpart_ind;  // F partition, coarse points by their rows' owners
    fpart.s = flo;
    cpart_ind.s = clo;
    struct Blk {
      Csr aff, affg, afc, acf, af;
      DBuf<int32_t> f2f;
    };
    std::vector<Blk> bk(P);
    each(d, [&](int r) {
      const int n = (int)V.rk[r].own;
      const int64_t nfo = nfr[r], nco = held.cnt(r) - nfr[r];
      DBuf<int32_t> ff(c, (size_t)std::max<int64_t>(1, nfo)), fc(c, (size_t)std::max<int64_t>(1, nfo)),
          cf(c, (size_t)std::max<int64_t>(1, nco)), af(c, (size_t)std::max<int64_t>(1, nfo));
      if (n)
        LAUNCH(c, k_blk_count, blocks_for(n, 256), 256, 0, n, loc[r].rp.p, loc[r].ci.p, ci[r].kind.p, flo[r], clo[r],
               ff.p, fc.p, cf.p);
      if (nfo) LAUNCH(c, k_add2, blocks_for(nfo, 256), 256, 0, nfo, ff.p, fc.p, af.p);
      auto fin = [&](Csr& m, int64_t rows, int64_t cols, const int32_t* cnt) {
        m = Csr();
        m.n = (int32_t)rows;
        m.m = (int32_t)cols;
        m.rp.alloc(c, (size_t)rows + 1);
        m.nnz = rows ? exclusive_scan(c, cnt, m.rp.p, rows) : 0;
        if (!rows) m.rp.zero(c);
        m.ci.alloc(c, (size_t)m.nnz);
        m.v.alloc(c, (size_t)m.nnz);
      };
      Blk& B = bk[r];
      fin(B.aff, nfo, nf, ff.p);
      fin(B.affg, nfo, n_cur, ff.p);
      fin(B.afc, nfo, nc, fc.p);
      fin(B.acf, nco, nf, cf.p);
      fin(B.af, nfo, n_cur, af.p);
      B.f2f.alloc(c, (size_t)std::max<int64_t>(1, nfo));
      if (n)
        LAUNCH(c, k_blk_fill, blocks_for(n, 256), 256, 0, n, loc[r].rp.p, loc[r].ci.p, loc[r].v.p, ci[r].kind.p,
               ci[r].gid.p, flo[r], clo[r], B.aff.rp.p, B.aff.ci.p, B.affg.ci.p, B.aff.v.p, B.affg.v.p, B.afc.rp.p,
               B.afc.ci.p, B.afc.v.p, B.acf.rp.p, B.acf.ci.p, B.acf.v.p, B.af.rp.p, B.af.ci.p, B.af.v.p, B.f2f.p);
    });
    {
      std::vector<int64_t> a(P, 0), b(P, 0), e(P, 0);
      each(d, [&](int r) {
        a[r] = bk[r].aff.nnz;
        b[r] = bk[r].afc.nnz;
        e[r] = bk[r].acf.nnz;
      });
      S.nnz_ff = sum_over_ranks(c, d, a);
      S.nnz_fc = sum_over_ranks(c, d, b);
      S.nnz_cf = sum_over_ranks(c, d, e);
      // theta of the final A_ff rows (air.cpp:355), max over the ranks
      std::vector<double> th((size_t)P, 0.0);
      each(d, [&](int r) {
        if (bk[r].aff.n) th[r] = dominance_max(c, bk[r].aff, (int)flo[r]);
      });
      allgather(c, d, th, 1);
      S.max_theta_post = 0.0;
      for (double x : th) S.max_theta_post = std::max(S.max_theta_post, x);
      if (!cfg.ddc_enabled) S.max_theta_pre = S.max_theta_post;
    }

    // ---- Aff^-1: F-space halo (VF), A_ff halo rows, the sorted ext layout
    DVec VF;
    VF.part = fpart;
    VF.N = nf;
    VF.rk.resize(P);
    each(d, [&](int r) { plan_rank(c, VF, r, {&bk[r].aff}); });
    finalize(c, VF, d, false);
    std::vector<FfRank> fr(P);
    std::vector<Csr> affc(P);
    std::vector<Csr> aff_rows(P);
    std::vector<DBuf<int32_t>> want(P);
    std::vector<int64_t> nw(P, 0);
    each(d, [&](int r) {
      csr_copy(c, bk[r].aff, affc[r]);
      to_layout(c, affc[r], VF, r, 0);
      csr_copy(c, bk[r].aff, aff_rows[r]);
      nw[r] = VF.rk[r].nhalo;
      want[r].view(VF.rk[r].halo.p, (size_t)std::max<int64_t>(1, nw[r]));
    });
    std::vector<Csr> aff_halo;
    fetch_rows(c, d, fpart, aff_rows, nf, want, nw, aff_halo);
    each(d, [&](int r) {
      const DVec::Rank& R = VF.rk[r];
      const std::vector<int64_t>& H = R.halo_host;
      const int64_t nb = std::lower_bound(H.begin(), H.end(), R.lo) - H.begin();
      fr[r].nb = nb;
      concat_rows(c, {&aff_halo[r], &bk[r].aff, &aff_halo[r]}, {{0, nb}, {0, R.own}, {nb, R.nhalo}}, nf, fr[r].ext);
      to_layout(c, fr[r].ext, VF, r, nb);
    });
    DistInverse inv;
    if (inj) {
      if (built >= (int64_t)inj->level_coeffs.size()) throw InvalidArgument("setup: injection table too short");
      inv = dist_checked_inverse(c, d, VF, fr, affc, cfg.poly_order, level_seed, &inj->level_coeffs[built],
                                 inj->level_eff[built]);
    } else {
      inv = dist_checked_inverse(c, d, VF, fr, affc, cfg.poly_order, level_seed, nullptr, 0);
    }
    S.coeffs = inv.coeffs;
    S.eff = inv.eff;
    S.growth = inv.growth;
    S.attempts = inv.attempts;
    {
      std::vector<int64_t> a(P, 0);
      each(d, [&](int r) { a[r] = inv.q[r].nnz; });
      S.nnz_ffinv = sum_over_ranks(c, d, a);
    }

    // ---- Aff^-1 with fine columns (Z's column space): the fine index of
    // every F number in A_ff's rows (own F rows and the F halo)
    std::vector<Csr> qfine(P);
    each(d, [&](int r) {
      const DVec::Rank& R = VF.rk[r];
      DBuf<int32_t> fmap(c, (size_t)std::max<int64_t>(1, nf)), hf(c, (size_t)std::max<int64_t>(1, R.nhalo));
      if (bk[r].aff.nnz)
        LAUNCH(c, k_scatter_fine, blocks_for(bk[r].aff.nnz, 256), 256, 0, bk[r].aff.nnz, bk[r].aff.ci.p,
               bk[r].affg.ci.p, fmap.p);
      if (R.nhalo) LAUNCH(c, k_gather_i32, blocks_for(R.nhalo, 256), 256, 0, R.nhalo, R.halo.p, fmap.p, hf.p);
      csr_copy(c, inv.q[r], qfine[r]);
      to_layout(c, qfine[r], VF, r, 0);
      if (qfine[r].nnz)
        LAUNCH(c, k_from_layout, blocks_for(qfine[r].nnz, 256), 256, 0, qfine[r].nnz, qfine[r].ci.p, bk[r].f2f.p,
               R.own, hf.p, (int64_t)0);
      qfine[r].m = (int32_t)n_cur;
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });

    // ---- Z = A_cf Aff^-1 (distance-2 rows of Aff^-1), R = [Z | I]
    DVec VZ;  // F-space halo of A_cf's columns
    VZ.part = fpart;
    VZ.N = nf;
    VZ.rk.resize(P);
    each(d, [&](int r) { plan_rank(c, VZ, r, {&bk[r].acf}); });
    std::vector<Csr> q_halo, r_rows(P);
    each(d, [&](int r) {
      nw[r] = VZ.rk[r].nhalo;
      want[r].view(VZ.rk[r].halo.p, (size_t)std::max<int64_t>(1, nw[r]));
    });
    fetch_rows(c, d, fpart, qfine, n_cur, want, nw, q_halo);
    each(d, [&](int r) {
      const DVec::Rank& R = VZ.rk[r];
      Csr bext, acfc, z;
      concat_rows(c, {&qfine[r], &q_halo[r]}, {{0, R.own}, {0, R.nhalo}}, n_cur, bext);
      csr_copy(c, bk[r].acf, acfc);
      to_layout(c, acfc, VZ, r, 0);
      spgemm(c, acfc, bext, z, cfg.drop_restrict, /*keep_diag=*/false);  // air.cpp:298-299
      // the C rows' own fine indices
      const int64_t nco = held.cnt(r) - nfr[r];
      DBuf<int32_t> c2f(c, (size_t)std::max<int64_t>(1, nco));
      {
        // own C rows in row order: gid of the rows whose kind < 0
        std::vector<int32_t> kind_h((size_t)V.rk[r].own);
        to_host(c, kind_h.data(), ci[r].kind.p, kind_h.size());
        std::vector<int32_t> cf_h;
        cf_h.reserve((size_t)nco);
        for (int64_t i = 0; i < V.rk[r].own; ++i)
          if (kind_h[i] < 0) cf_h.push_back((int32_t)(held.lo(r) + i));
        to_device(c, c2f.p, cf_h.data(), cf_h.size());
      }
      restriction_from_z(c, z, nullptr, c2f.p, n_cur, r_rows[r]);
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });
    {
      std::vector<int64_t> a(P, 0);
      each(d, [&](int r) { a[r] = r_rows[r].nnz; });
      S.nnz_r = sum_over_ranks(c, d, a);
    }

    // ---- one-point P (own rows), its halo entries, A P
    std::vector<DBuf<int32_t>> pmap(P);
    std::vector<Csr> ap(P);
    each(d, [&](int r) {
      DVec::Rank& R = V.rk[r];
      pmap[r].alloc(c, (size_t)std::max<int64_t>(1, R.own));
      prolongation_map_fused(c, ci[r].label.p, ci[r].cnum.p, loc[r], cfg.strength_alpha, pmap[r].p);
      if (R.own) LAUNCH(c, k_i2d, blocks_for(R.own, 256), 256, 0, R.own, pmap[r].p, R.buf.p);
    });
    exchange(c, d, V);
    {
      std::vector<int64_t> a(P, 0);
      each(d, [&](int r) {
        DBuf<unsigned long long> k(c, 1);
        k.zero(c);
        const int64_t n = V.rk[r].own;
        if (n) LAUNCH(c, k_count_ge0, blocks_for(n, 256), 256, 0, n, pmap[r].p, k.p);
        a[r] = (int64_t)read1(c, k.p);
      });
      S.nnz_p = sum_over_ranks(c, d, a);
    }
    each(d, [&](int r) {
      DVec::Rank& R = V.rk[r];
      const int64_t t = R.own + R.nhalo;
      DBuf<int32_t> pm(c, (size_t)std::max<int64_t>(1, t));
      if (t) LAUNCH(c, k_d2i, blocks_for(t, 256), 256, 0, t, R.buf.p, pm.p);
      Csr pext;
      prolongation_from_map(c, pm.p, (int)t, (int)nc, pext);
      spgemm(c, loc[r], pext, ap[r]);  // air.cpp:268-271 (A P, nothing dropped)
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });

    // ---- the fast V-cycle's fused operators on the own F rows (fused.cu,
    // same products in the same order as one GPU, so the same bits):
    // A_F P = the F rows of A P; W_2 = (Q + Q) - (Q A_ff) Q with Q A_ff from
    // A_ff's F-halo rows and (Q A_ff) Q from the distance-2 rows of Q
    std::vector<Csr> afp(P), wk(P);
    const int64_t fsm = cfg.fused_smooths;
    const bool fused = fsm >= 0 && fsm <= 2;
    if (fused) {
      each(d, [&](int r) {
        const int64_t nfo = nfr[r];
        select_rows(c, ap[r], held.lo(r), bk[r].f2f.p, nfo, afp[r]);
        afp[r].m = (int32_t)nc;
      });
      std::vector<Csr> u(P);
      if (fsm == 2) {
        each(d, [&](int r) {
          Csr qv, bext;
          csr_copy(c, inv.q[r], qv);
          to_layout(c, qv, VF, r, 0);
          concat_rows(c, {&bk[r].aff, &aff_halo[r]}, {{0, VF.rk[r].own}, {0, VF.rk[r].nhalo}}, nf, bext);
          spgemm(c, qv, bext, u[r]);  // Q A_ff, global F columns
          CUDA_CHECK(cudaStreamSynchronize(c.stream));
        });
      }
      DVec VW;  // F-space halo of Q A_ff's columns (distance 2)
      VW.part = fpart;
      VW.N = nf;
      VW.rk.resize(P);
      std::vector<Csr> q2;
      if (fsm == 2) {
        each(d, [&](int r) {
          plan_rank(c, VW, r, {&u[r]});
          nw[r] = VW.rk[r].nhalo;
          want[r].view(VW.rk[r].halo.p, (size_t)std::max<int64_t>(1, nw[r]));
        });
        fetch_rows(c, d, fpart, inv.q, nf, want, nw, q2);
      }
      each(d, [&](int r) {
        if (fsm == 0) {  // no F-smooth: an empty W
          wk[r] = Csr();
          wk[r].n = (int32_t)nfr[r];
          wk[r].m = (int32_t)nf;
          wk[r].rp.alloc(c, (size_t)nfr[r] + 1);
          wk[r].rp.zero(c);
          return;
        }
        Csr w1;
        csr_add(c, 1.0, inv.q[r], 0.0, inv.q[r], w1);  // W_1 = Q
        if (fsm == 1) {
          wk[r] = std::move(w1);
          return;
        }
        Csr bext, uv, waq, qw;
        concat_rows(c, {&inv.q[r], &q2[r]}, {{0, VW.rk[r].own}, {0, VW.rk[r].nhalo}}, nf, bext);
        csr_copy(c, u[r], uv);
        to_layout(c, uv, VW, r, 0);
        spgemm(c, uv, bext, waq);
        csr_add(c, 1.0, inv.q[r], 1.0, w1, qw);
        csr_add(c, 1.0, qw, -1.0, waq, wk[r]);
        CUDA_CHECK(cudaStreamSynchronize(c.stream));
      });
      std::vector<int64_t> a(P, 0), b(P, 0);
      each(d, [&](int r) {
        a[r] = afp[r].nnz;
        b[r] = wk[r].nnz;
      });
      D.nnz_afp = sum_over_ranks(c, d, a);
      D.nnz_w = sum_over_ranks(c, d, b);
    }

    // ---- R (A P) from the A P halo rows (distance 2), full diagonal
    DVec VR;  // fine-space halo of R's columns
    VR.part = held;
    VR.N = n_cur;
    VR.rk.resize(P);
    each(d, [&](int r) { plan_rank(c, VR, r, {&r_rows[r]}); });
    std::vector<Csr> ap_halo, next(P);
    each(d, [&](int r) {
      nw[r] = VR.rk[r].nhalo;
      want[r].view(VR.rk[r].halo.p, (size_t)std::max<int64_t>(1, nw[r]));
    });
    fetch_rows(c, d, held, ap, nc, want, nw, ap_halo);
    each(d, [&](int r) {
      const DVec::Rank& R = VR.rk[r];
      Csr bext, rc, rap;
      concat_rows(c, {&ap[r], &ap_halo[r]}, {{0, R.own}, {0, R.nhalo}}, nc, bext);
      csr_copy(c, r_rows[r], rc);
      to_layout(c, rc, VR, r, 0);
      spgemm(c, rc, bext, rap, cfg.drop_coarse, /*keep_diag=*/true, nullptr, (int)clo[r], nc);
      with_full_diagonal(c, rap, next[r], (int)clo[r], true);
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
    });

    // ---- pieces of this level for the solve
    pc.lv.emplace_back();
    pc.lv.back().resize(P);
    pc.fpart.push_back(fpart);
    pc.n.push_back(n_cur);
    pc.nf.push_back(nf);
    each(d, [&](int r) {
      DistPieces::LevelRank& L = pc.lv.back()[r];
      L.AF = std::move(bk[r].af);
      L.AFFG = std::move(bk[r].affg);
      L.FINV = std::move(inv.q[r]);
      if (fused) {
        L.AFP = std::move(afp[r]);
        L.W = std::move(wk[r]);
      }
      L.pmap = std::move(pmap[r]);
      L.f2f = std::move(bk[r].f2f);
    });
    pending_r = std::move(r_rows);
    pending_r.resize(P);
    pending_part = cpart_ind;
    d.lv.push_back(std::move(D));
    d.summary.push_back(S);
    // ---- next level
    cur = std::move(next);
    cur.resize(P);
    held = cpart_ind;
    n_cur = nc;
  }
  // coarsest grid on rank 0
  const int64_t L = (int64_t)d.lv.size();
  if (!coarse_valid) {
    auto [ci, qnnz] = coarse_try(L);
    coarse = std::move(ci);
    coarse_inv_nnz = qnnz;
  }
  {
    const Part g0 = gathered(n_cur, P);
    std::vector<int64_t> nz(P, 0);
    each(d, [&](int r) { nz[r] = cur[r].nnz; });
    const int64_t coarse_nnz = sum_over_ranks(c, d, nz);
    migrate(c, d, held, g0, cur, n_cur);
    if (L) {
      migrate(c, d, pending_part, g0, pending_r, pc.n.back());
      each(d, [&](int r) { pc.lv.back()[r].R = std::move(pending_r[r]); });
    }
    pc.coarse_n = n_cur;
    pc.fused_smooths = (cfg.fused_smooths >= 0 && cfg.fused_smooths <= 2) ? cfg.fused_smooths : -1;
    pc.AC.resize(P);
    pc.ACI.resize(P);
    pc.A0.resize(P);
    each(d, [&](int r) {
      if (r == 0) {
        pc.AC[0] = std::move(cur[0]);
        pc.ACI[0] = std::move(coarse.q);
      } else {
        empty_rows(c, pc.AC[r], n_cur);
        empty_rows(c, pc.ACI[r], n_cur);
      }
      pc.A0[r] = std::move(top[r]);
    });
    if (L == 0) {  // no fine level: the top operator is the coarse grid (gathered)
      each(d, [&](int r) {
        if (r == 0)
          csr_copy(c, pc.AC[0], pc.A0[0]);
        else
          empty_rows(c, pc.A0[r], n_cur);
      });
    }
    DHier::Summary S;
    S.n = n_cur;
    S.nnz = coarse_nnz;
    S.nnz_ffinv = coarse_inv_nnz;
    S.coeffs = coarse.coeffs;
    S.eff = coarse.eff;
    S.attempts = coarse.attempts;
    S.growth = coarse.growth;
    d.summary.push_back(S);
  }
  dist_build(c, d, pc);
  d.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace airg
