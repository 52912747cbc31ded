// Row-slab distributed AIRG solve (see dist.cuh).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <cstring>

#include "dist.cuh"
#include "fusedx.cuh"
#include "gmres.cuh"
#include "tiled.cuh"

namespace airg {

int Part::owner(int64_t g) const {
  return (int)(std::upper_bound(s.begin(), s.end(), g) - s.begin()) - 1;
}

namespace {

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ int owner_of(const int64_t* __restrict__ s, int P, int64_t g) {
  int lo = 0, hi = P;  // largest r with s[r] <= g (and non-empty ranges win)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void k_locality(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const int64_t* __restrict__ s, int P,
                           unsigned long long* __restrict__ cnt) {  // [2P]: local, nonlocal
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = owner_of(s, P, i);
  unsigned long long loc = 0, non = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) (owner_of(s, P, ci[k]) == r ? loc : non)++;
  if (loc) atomicAdd(cnt + r, loc);
  if (non) atomicAdd(cnt + P + r, non);
}

__global__ void k_slice(int n_local, int64_t row0, const int32_t* __restrict__ rp,
                        const int32_t* __restrict__ ci, const double* __restrict__ v,
                        int32_t* __restrict__ orp, int32_t* __restrict__ oci,
                        double* __restrict__ ov) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n_local) return;
  const int base = rp[row0];
  orp[i] = rp[row0 + i] - base;
  if (i == n_local) return;
  for (int k = rp[row0 + i]; k < rp[row0 + i + 1]; ++k) {
    oci[k - base] = ci[k];
    ov[k - base] = v[k];
  }
}

__global__ void k_mark_cols(int64_t nnz, const int32_t* __restrict__ ci, int64_t lo, int64_t hi,
                            int32_t* __restrict__ mark) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int64_t c = ci[k] & 0x7fffffff;
  if (c < lo || c >= hi) mark[c] = 1;
}
__global__ void k_mark_vals(int64_t n, const int32_t* __restrict__ idx, int64_t lo, int64_t hi,
                            int32_t* __restrict__ mark) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t c = idx[k];
  if (c >= 0 && (c < lo || c >= hi)) mark[c] = 1;
}
__global__ void k_compact(int64_t N, const int32_t* __restrict__ mark, const int32_t* __restrict__ pos,
                          int32_t* __restrict__ out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < N && mark[g]) out[pos[g]] = (int32_t)g;
}
__global__ void k_src(int64_t nh, const int32_t* __restrict__ halo, const int64_t* __restrict__ s, int P,
                      int32_t* __restrict__ src_rank, int32_t* __restrict__ src_idx) {
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= nh) return;
  const int r = owner_of(s, P, halo[h]);
  src_rank[h] = r;
  src_idx[h] = (int32_t)(halo[h] - s[r]);
}
__device__ __forceinline__ int32_t remap_one(int64_t c, int64_t lo, int64_t hi, int64_t own,
                                             const int32_t* __restrict__ halo, int64_t nh) {
  if (c >= lo && c < hi) return (int32_t)(c - lo);
  int64_t a = 0, b = nh;
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (halo[m] < c)
      a = m + 1;
    else
      b = m;
  }
  return (int32_t)(own + a);
}
__global__ void k_remap_cols(int64_t nnz, int32_t* __restrict__ ci, int64_t lo, int64_t hi, int64_t own,
                             const int32_t* __restrict__ halo, int64_t nh) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int32_t raw = ci[k];
  const int32_t flag = raw & (int32_t)0x80000000;
  ci[k] = remap_one(raw & 0x7fffffff, lo, hi, own, halo, nh) | flag;
}
__global__ void k_remap_vals(int64_t n, const int32_t* __restrict__ in, int32_t* __restrict__ out,
                             int64_t lo, int64_t hi, int64_t own, const int32_t* __restrict__ halo,
                             int64_t nh) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = in[k] < 0 ? -1 : remap_one(in[k], lo, hi, own, halo, nh);
}
__global__ void k_shift(int64_t n, const int32_t* __restrict__ in, int64_t off, int32_t* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = (int32_t)(in[k] - off);
}
// count of sorted[] entries < bound[j]  (F points below each slab boundary)
__global__ void k_count_below(const int32_t* __restrict__ sorted, int64_t n, const int64_t* __restrict__ bound,
                              int nb, int64_t* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  int64_t a = 0, b = n;
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (sorted[m] < bound[j])
      a = m + 1;
    else
      b = m;
  }
  out[j] = a;
}

// halo exchange kernels
__global__ void k_gather_halo(int64_t nh, const int32_t* __restrict__ src_rank,
                              const int32_t* __restrict__ src_idx, double* const* __restrict__ bases,
                              double* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h < nh) dst[h] = bases[src_rank[h]][src_idx[h]];
}
__global__ void k_pack(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                       double* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = src[idx[k]];
}

// solve kernels (local versions of solve.cu's)
// four rows per thread (int4 map load, double2 stores); the owned slices
// start at the buffers' bases, 16-byte aligned
__device__ __forceinline__ double prolong_one_l(int j, const double* __restrict__ ec) {
  const double pe = j >= 0 ? __dadd_rn(0.0, __dmul_rn(1.0, ec[j])) : 0.0;
  return __dadd_rn(0.0, __dmul_rn(1.0, pe));
}
__global__ void k_prolong4_l(int n, const int32_t* __restrict__ pmap, const double* __restrict__ ec,
                             double* __restrict__ x) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int n4 = n >> 2;
  int4 j = make_int4(-1, -1, -1, -1);
  if (q < n4) j = __ldg(reinterpret_cast<const int4*>(pmap) + q);
  pdl_wait();
  pdl_trigger();
  if (q == n4) {
    for (int i = 4 * n4; i < n; ++i) x[i] = prolong_one_l(__ldg(pmap + i), ec);
    return;
  }
  if (q > n4) return;
  double2* x2 = reinterpret_cast<double2*>(x);
  x2[2 * q] = make_double2(prolong_one_l(j.x, ec), prolong_one_l(j.y, ec));
  x2[2 * q + 1] = make_double2(prolong_one_l(j.z, ec), prolong_one_l(j.w, ec));
}
__global__ void k_axpy1_l(int n, const double* __restrict__ e, double* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;  // two entries per thread
  const int n2 = n >> 1;
  if (q < n2) {
    const double2 ev = reinterpret_cast<const double2*>(e)[q];
    double2 xv = reinterpret_cast<double2*>(x)[q];
    xv.x = __dadd_rn(xv.x, __dmul_rn(1.0, ev.x));
    xv.y = __dadd_rn(xv.y, __dmul_rn(1.0, ev.y));
    reinterpret_cast<double2*>(x)[q] = xv;
  } else if (q == n2 && (n & 1)) {
    x[n - 1] = __dadd_rn(x[n - 1], __dmul_rn(1.0, e[n - 1]));
  }
}
__global__ void k_sum(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double sm[32];
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
  }
}

// epilogues (local layouts)
struct LStore {
  double* y;
  __device__ void row(int r, double acc) const { y[r] = acc; }
  __device__ void finish() const {}
};
struct LFres1 {
  const double* b;
  const int32_t* f2f;
  double* rf;
  double* sc;
  // operands written two or more kernels back, loaded before the PDL wait
  // (solve.cu explains the rule; halo exchanges in between only add order)
  struct Pre {
    double bb;
  };
  __device__ Pre pre(int k) const { return Pre{b[f2f[k]]}; }
  __device__ void row2_pre(int k, double sf, double s, const Pre& p) const {
    sc[k] = s;
    rf[k] = __dsub_rn(__dsub_rn(p.bb, sf), s);
  }
};
struct LFres2 {
  const double* b;
  const int32_t* f2f;
  const double* sc;
  double* rf;
  __device__ void finish() const {}
  struct Pre {
    double bb, s;
  };
  __device__ Pre pre(int k) const { return Pre{b[f2f[k]], sc[k]}; }
  __device__ void row_pre(int k, double sf, const Pre& p) const { rf[k] = __dsub_rn(__dsub_rn(p.bb, sf), p.s); }
};
struct LFupd {
  const int32_t* f2f;
  double* x;
  __device__ void finish() const {}
  struct Pre {
    int i;
    double x0;
  };
  __device__ Pre pre(int k) const {
    const int i = f2f[k];
    return Pre{i, x[i]};
  }
  __device__ void row_pre(int, double d, const Pre& p) const { x[p.i] = __dadd_rn(p.x0, d); }
};
struct LCres {
  const double* rhs;
  double* r;
  __device__ void finish() const {}
  struct Pre {
    double rr;
  };
  __device__ Pre pre(int i) const { return Pre{rhs[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const { r[i] = __dsub_rn(p.rr, acc); }
};
struct LCupd {
  double* e;
  int first;
  __device__ void finish() const {}
  struct Pre {
    double e0;
  };
  __device__ Pre pre(int i) const { return Pre{first ? 0.0 : e[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const { e[i] = __dadd_rn(p.e0, __dmul_rn(1.0, acc)); }
};
struct LResid {
  const double* b;
  double* r;
  double* part;
  mutable double s;
  struct Pre {  // the right-hand side is constant during the solve
    double bb;
  };
  __device__ Pre pre(int i) const { return Pre{b[i]}; }
  __device__ void row_pre(int i, double acc, const Pre& p) const {
    const double ri = __dsub_rn(p.bb, acc);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  __device__ void finish() const {
    __shared__ double sm[32];  // any block size up to 1024 (SELL launches 256)
    double v = s;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
  }
};

// fast V-cycle: r1 = b_F - (A_F P) e_c (solve.cu EpiFres1P)
struct LFres1P {
  const double* b;
  const int32_t* f2f;
  double* rf;
  __device__ void finish() const {}
  struct Pre {
    double bb;
  };
  __device__ Pre pre(int k) const { return Pre{b[f2f[k]]}; }
  __device__ void row_pre(int k, double acc, const Pre& p) const { rf[k] = p.bb - acc; }
};

// exact thread-per-row kernels in the batch kind of the matrix (tiled.cuh);
// fast: lane groups, FMA, tree sums
template <class Epi>
void launch_rows(Ctx& c, const Csr& m, const double* x, const Epi& epi, bool fast = false) {
  LAUNCH_ROWS_MODE(c, Epi, tview(m), x, epi, fast);
}
template <class Epi>
void launch_rows_fc(Ctx& c, const Csr& m, const double* x, const Epi& epi) {
  LAUNCH_ROWS_FC_MODE(c, Epi, tview(m), x, epi, false);
}

}  // namespace

// ---- host helpers ---------------------------------------------------------------
// partition_rows (partition_model.cpp:8-22) on `active` logical ranks, logical
// rank k placed on physical rank k * stride
Part balanced(int64_t n, int active, int P) {
  const int ranks = (int)std::min<int64_t>(active, std::max<int64_t>(n, 1));
  const int stride = std::max(1, P / std::max(1, active));
  std::vector<int64_t> lstart(ranks + 1, 0);
  const int64_t base = n / ranks, extra = n % ranks;
  for (int k = 0; k < ranks; ++k) lstart[k + 1] = lstart[k] + base + (k < extra ? 1 : 0);
  Part p;
  p.s.assign(P + 1, n);
  for (int q = 0; q <= P; ++q) {
    // first logical block placed at a physical rank >= q
    int k = (q + stride - 1) / stride;
    p.s[q] = k < ranks ? lstart[k] : n;
  }
  p.s[0] = 0;
  p.s[P] = n;
  return p;
}

// merge adjacent logical pairs (r -> r / 2, partition_model.cpp:101-104)
Part merged(const Part& p, int active, int new_active) {
  const int P = p.P();
  const int stride_old = std::max(1, P / std::max(1, active));
  const int stride_new = std::max(1, P / std::max(1, new_active));
  // logical block k of the old partition starts at p.s[k * stride_old]
  std::vector<int64_t> lstart;
  for (int k = 0; k < active; ++k) lstart.push_back(p.s[std::min(P, k * stride_old)]);
  lstart.push_back(p.s[P]);
  std::vector<int64_t> ns(new_active + 1);
  for (int k = 0; k < new_active; ++k) ns[k] = lstart[std::min(active, 2 * k)];
  ns[new_active] = p.s[P];
  Part out;
  out.s.assign(P + 1, p.s[P]);
  for (int q = 0; q <= P; ++q) {
    int k = (q + stride_new - 1) / stride_new;
    out.s[q] = k < new_active ? ns[k] : p.s[P];
  }
  out.s[0] = 0;
  return out;
}

Part gathered(int64_t n, int P) {
  Part p;
  p.s.assign(P + 1, n);
  p.s[0] = 0;
  return p;
}

// mean over ranks of local / non-local nnz (partition_model.cpp:53-64)
// locality_ratio (partition_model.cpp:53-64) of a contiguous partition;
// share: local_share (:66-75), the global fraction of on-rank entries
double locality(Ctx& c, const Csr& a, const Part& p, double* share = nullptr) {
  const int P = p.P();
  if (share) *share = 1.0;
  if (a.n == 0) return INFINITY;
  DBuf<int64_t> ds(c, (size_t)P + 1);
  to_device(c, ds.p, p.s.data(), (size_t)P + 1);
  DBuf<unsigned long long> cnt(c, (size_t)2 * P);
  cnt.zero(c);
  LAUNCH(c, k_locality, blocks_for(a.n, 256), 256, 0, a.n, a.rp.p, a.ci.p, ds.p, P, cnt.p);
  std::vector<unsigned long long> h(2 * P);
  to_host(c, h.data(), cnt.p, h.size());
  double sum = 0.0;
  int contributing = 0;
  unsigned long long loc = 0, tot = 0;
  for (int r = 0; r < P; ++r) {
    loc += h[r];
    tot += h[r] + h[P + r];
    if (h[P + r] == 0) continue;
    sum += (double)h[r] / (double)h[P + r];
    ++contributing;
  }
  if (share && tot) *share = (double)loc / (double)tot;
  return contributing ? sum / contributing : INFINITY;
}

void slice(Ctx& c, const Csr& a, int64_t lo, int64_t hi, Csr& out) {
  const int64_t n = hi - lo;
  int32_t b[2] = {0, 0};
  if (n > 0) {
    to_host(c, &b[0], a.rp.p + lo, 1);
    to_host(c, &b[1], a.rp.p + hi, 1);
  }
  out.alloc(c, n, a.m, b[1] - b[0]);
  if (n > 0)
    LAUNCH(c, k_slice, blocks_for(n + 1, 256), 256, 0, (int)n, lo, a.rp.p, a.ci.p, a.v.p, out.rp.p,
           out.ci.p, out.v.p);
  else
    out.rp.zero(c);
}

void Marks::init(Ctx& c, int64_t n) {
  N = n;
  m.alloc(c, (size_t)std::max<int64_t>(1, n));
  m.zero(c);
}
void Marks::cols(Ctx& c, const Csr& a, int64_t lo, int64_t hi) {
  if (a.nnz) LAUNCH(c, k_mark_cols, blocks_for(a.nnz, 256), 256, 0, a.nnz, a.ci.p, lo, hi, m.p);
}
void Marks::vals(Ctx& c, const int32_t* idx, int64_t n, int64_t lo, int64_t hi) {
  if (n) LAUNCH(c, k_mark_vals, blocks_for(n, 256), 256, 0, n, idx, lo, hi, m.p);
}

void set_halo(Ctx& c, DVec& V, int r, Marks& mk) {
  DVec::Rank& R = V.rk[r];
  R.own = V.part.cnt(r);
  R.lo = V.part.lo(r);
  DBuf<int32_t> pos(c, (size_t)V.N + 1);
  const int64_t nh = V.N ? exclusive_scan(c, mk.m.p, pos.p, V.N) : 0;
  R.nhalo = nh;
  R.halo.alloc(c, (size_t)std::max<int64_t>(1, nh));
  if (V.N) LAUNCH(c, k_compact, blocks_for(V.N, 256), 256, 0, V.N, mk.m.p, pos.p, R.halo.p);
  std::vector<int32_t> hh((size_t)nh);
  to_host(c, hh.data(), R.halo.p, (size_t)nh);
  R.halo_host.assign(hh.begin(), hh.end());
}

// One rank per process, each knowing only its own halo: the halo lists of
// all ranks all-gathered (sizes, then the padded lists), so every process
// derives its send lists (and p2p push plans) as in the all-ranks plan.
void share_halos(Ctx& c, const DHier& d, DVec& V) {
  const int P = V.part.P(), me = d.me;
  DVec::Rank& M = V.rk[me];
  DBuf<int64_t> mine(c, 1), sz(c, (size_t)P);
  to_device(c, mine.p, &M.nhalo, 1);
  NCCL_CHECK(ncclAllGather(mine.p, sz.p, 1, ncclInt64, d.comm, c.stream));
  std::vector<int64_t> hs(P);
  to_host(c, hs.data(), sz.p, (size_t)P);
  const int64_t mx = std::max<int64_t>(1, *std::max_element(hs.begin(), hs.end()));
  DBuf<int32_t> send(c, (size_t)mx), all(c, (size_t)mx * P);
  if (M.nhalo)
    CUDA_CHECK(cudaMemcpyAsync(send.p, M.halo.p, sizeof(int32_t) * M.nhalo, cudaMemcpyDeviceToDevice, c.stream));
  NCCL_CHECK(ncclAllGather(send.p, all.p, (size_t)mx, ncclInt32, d.comm, c.stream));
  std::vector<int32_t> h((size_t)mx * P);
  to_host(c, h.data(), all.p, h.size());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    DVec::Rank& Q = V.rk[q];
    Q.own = V.part.cnt(q);
    Q.lo = V.part.lo(q);
    Q.nhalo = hs[q];
    Q.halo_host.assign(h.begin() + (size_t)q * mx, h.begin() + (size_t)q * mx + hs[q]);
  }
}

// After every rank's halo is known: buffers, emulation tables, NCCL lists.
void finalize(Ctx& c, DVec& V, const DHier& d, bool peers_known) {
  const int P = V.part.P();
  if (!peers_known && d.me >= 0 && P > 1) share_halos(c, d, V);
  DBuf<int64_t> ds(c, (size_t)P + 1);
  to_device(c, ds.p, V.part.s.data(), (size_t)P + 1);
  std::vector<double*> bases(P, nullptr);
  for (int r = 0; r < P; ++r) {
    DVec::Rank& R = V.rk[r];
    R.recv_off.assign(P, 0);
    R.recv_cnt.assign(P, 0);
    for (int64_t g : R.halo_host) R.recv_cnt[V.part.owner(g)]++;
    for (int q = 1; q < P; ++q) R.recv_off[q] = R.recv_off[q - 1] + R.recv_cnt[q - 1];
    if (!d.mine(r)) continue;
    R.buf.alloc(c, (size_t)std::max<int64_t>(1, R.own + R.nhalo));
    R.buf.zero(c);
    bases[r] = R.buf.p;
    if (d.me < 0 && R.nhalo) {
      R.src_rank.alloc(c, (size_t)R.nhalo);
      R.src_idx.alloc(c, (size_t)R.nhalo);
      LAUNCH(c, k_src, blocks_for(R.nhalo, 256), 256, 0, R.nhalo, R.halo.p, ds.p, P, R.src_rank.p,
             R.src_idx.p);
    }
  }
  if (d.me >= 0) {  // my send lists: the entries of every peer's halo that I own
    DVec::Rank& M = V.rk[d.me];
    std::vector<int32_t> idx;
    M.send_off.assign(P, 0);
    M.send_cnt.assign(P, 0);
    for (int q = 0; q < P; ++q) {
      M.send_off[q] = (int64_t)idx.size();
      if (q == d.me) continue;
      for (int64_t g : V.rk[q].halo_host)
        if (g >= M.lo && g < M.lo + M.own) idx.push_back((int32_t)(g - M.lo));
      M.send_cnt[q] = (int64_t)idx.size() - M.send_off[q];
    }
    M.send_idx.alloc(c, std::max<size_t>(1, idx.size()));
    to_device(c, M.send_idx.p, idx.data(), idx.size());
    M.send_buf.alloc(c, std::max<size_t>(1, idx.size()));
  } else {
    V.bases.alloc(c, (size_t)P);
    to_device(c, V.bases.p, bases.data(), (size_t)P);
  }
}

void remap(Ctx& c, Csr& a, const DVec& V, int r) {
  const DVec::Rank& R = V.rk[r];
  if (a.nnz)
    LAUNCH(c, k_remap_cols, blocks_for(a.nnz, 256), 256, 0, a.nnz, a.ci.p, R.lo, R.lo + R.own, R.own,
           R.halo.p, R.nhalo);
  a.m = (int32_t)(R.own + R.nhalo);
}

// halo exchange of one vector (all local ranks)
void exchange(Ctx& c, DHier& d, DVec& V) {
  if (d.p2p.on && V.slot >= 0) {
    p2p_exchange(c, d, V);
    return;
  }
  const int P = V.part.P();
  if (d.me < 0) {
    for (int r = 0; r < P; ++r) {
      DVec::Rank& R = V.rk[r];
      if (R.nhalo)
        LAUNCH_PDL(c, k_gather_halo, blocks_for(R.nhalo, 256), 256, 0, R.nhalo, R.src_rank.p,
                   R.src_idx.p, (double* const*)V.bases.p, R.buf.p + R.own);
    }
    return;
  }
  if (P == 1) return;  // a single rank has no halo
  DVec::Rank& M = V.rk[d.me];
  const int64_t ns = M.send_off[P - 1] + M.send_cnt[P - 1];
  if (ns) LAUNCH_PDL(c, k_pack, blocks_for(ns, 256), 256, 0, ns, M.send_idx.p, M.buf.p, M.send_buf.p);
  bool any = ns > 0 || M.nhalo > 0;
  for (int q = 0; q < P && !any; ++q) any = M.send_cnt[q] || M.recv_cnt[q];
  // no traffic of mine: no peer sends to or receives from me either (a send
  // list is the owner's view of a peer's receive list), so no NCCL call
  if (!any) return;
  NCCL_CHECK(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == d.me) continue;
    if (M.send_cnt[q])
      NCCL_CHECK(ncclSend(M.send_buf.p + M.send_off[q], (size_t)M.send_cnt[q], ncclDouble, q, d.comm, c.stream));
    if (M.recv_cnt[q])
      NCCL_CHECK(ncclRecv(M.buf.p + M.own + M.recv_off[q], (size_t)M.recv_cnt[q], ncclDouble, q, d.comm,
                          c.stream));
  }
  NCCL_CHECK(ncclGroupEnd());
}

// the kernels that read V's halo since exchange(V) have been enqueued: the
// p2p transport hands the halo slots back to their owners (no-op otherwise)
void release(Ctx& c, DHier& d, DVec& V) {
  if (d.p2p.on && V.slot >= 0) p2p_release(c, d, V);
}

namespace {

// ---- distributed CF split kernels (local column indices into [own | halo]) ----
__device__ __forceinline__ uint64_t dsplitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ int64_t gidx(int32_t lc, int64_t lo, int64_t own, const int32_t* halo) {
  return lc < own ? lo + lc : (int64_t)halo[lc - own];
}
__global__ void k_dweights(int n, int64_t lo, const int32_t* __restrict__ s_cnt, const double* __restrict__ stb,
                           uint64_t key, double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t deg = (int64_t)s_cnt[i] + (int64_t)stb[i];
  const double u = (double)(dsplitmix(key ^ dsplitmix((uint64_t)(lo + i))) >> 11) * 0x1.0p-53;
  w[i] = __dadd_rn((double)deg, u);
}
__global__ void k_to_u8(int64_t n, const double* __restrict__ lab, uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint8_t)lab[i];
}
__global__ void k_scatter_add(int64_t nh, const int32_t* __restrict__ src_rank,
                              const int32_t* __restrict__ src_idx, double* const* __restrict__ bases,
                              const double* __restrict__ halo_vals) {
  const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (h < nh) atomicAdd(&bases[src_rank[h]][src_idx[h]], halo_vals[h]);
}
__global__ void k_unpack_add(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                             double* __restrict__ dst) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) atomicAdd(&dst[idx[k]], src[k]);
}

// ---- fused distributed split (same passes as cfsplit.cu's cf_split_fused) ----
__global__ void k_frows(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const double* __restrict__ v, double alpha, double* __restrict__ thr,
                        int32_t* __restrict__ s_cnt, double* __restrict__ stb,
                        unsigned long long* __restrict__ s_total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int cnt = 0;
  if (i < n) {
    double off_max = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] != i) off_max = fmax(off_max, fabs(v[k]));
    const double t = __dmul_rn(alpha, off_max);
    thr[i] = t;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const double mag = fabs(v[k]);
      if (ci[k] != i && mag > 0.0 && mag >= t) {
        ++cnt;
        atomicAdd(stb + ci[k], 1.0);
      }
    }
    s_cnt[i] = cnt;
  }
  block_add(s_total, (unsigned long long)cnt);
}
__global__ void k_fmarks(int n, int64_t lo, int64_t own, const int32_t* __restrict__ halo,
                         const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                         const double* __restrict__ v, const double* __restrict__ thr,
                         const double* __restrict__ w, double* __restrict__ nm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double wi = w[i], t = thr[i];
  const int64_t gi = lo + i;
  bool mine = false;
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int32_t lc = ci[k];
    const double mag = fabs(v[k]);
    if (lc == i || !(mag > 0.0) || !(mag >= t)) continue;
    const double wj = w[lc];
    const int64_t gj = gidx(lc, lo, own, halo);
    if (wj != wi ? wj < wi : gj < gi)  // weight_less(j, i)
      mine = true;
    else
      nm[lc] = 1.0;
  }
  if (mine) nm[i] = 1.0;
}
__global__ void k_flabels(int n, const double* __restrict__ w, const double* __restrict__ nm,
                          double* __restrict__ lab, unsigned long long* __restrict__ nf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (i < n) {
    f = w[i] < 1.0 || nm[i] == 0.0;
    lab[i] = f ? (double)AIRG_F : (double)AIRG_C;
  }
  block_add(nf, f ? 1ull : 0ull);
}
__global__ void k_ftheta(int n, int64_t lo, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                         const double* __restrict__ v, const double* __restrict__ lab, double* __restrict__ theta,
                         unsigned long long* __restrict__ maxbits, unsigned long long* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long tb = 0;
  if (i < n && lab[i] == (double)AIRG_F) {
    double off = 0.0, diag = 0.0;
    bool seen = false;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t lc = ci[k];
      if (lab[lc] != (double)AIRG_F) continue;
      if (lc == i) {
        diag = fabs(v[k]);
        seen = true;
      } else {
        off = __dadd_rn(off, fabs(v[k]));
      }
    }
    if (!seen || diag == 0.0) {
      atomicMin(bad, (unsigned long long)(lo + i));  // global fine row; F sub-index on the host
      theta[i] = 0.0;
    } else {
      const double t = __ddiv_rn(off, diag);
      theta[i] = t;
      tb = (unsigned long long)__double_as_longlong(t);
    }
  }
  block_max(maxbits, tb);
}
__global__ void k_fhist(int n, const double* __restrict__ lab, const double* __restrict__ theta,
                        const unsigned long long* __restrict__ maxbits, int64_t bins,
                        unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int sh[];
  const bool priv = bins <= 8192;
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const double mx = __longlong_as_double((long long)*maxbits);
  const double width = mx > 0.0 ? __ddiv_rn(mx, (double)bins) : 1.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (lab[i] != (double)AIRG_F) continue;
    int64_t b = (int64_t)__ddiv_rn(theta[i], width);
    if (b > bins - 1) b = bins - 1;
    if (priv)
      atomicAdd(sh + b, 1u);
    else
      atomicAdd(hist + b, 1ull);
  }
  __syncthreads();
  if (priv)
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
      if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
}
__global__ void k_fconvert(int n, const double* __restrict__ theta, const double* __restrict__ sel,
                           const unsigned long long* __restrict__ bad, double* __restrict__ lab,
                           unsigned long long* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool conv = false;
  if (i < n && *bad == ~0ull && lab[i] == (double)AIRG_F) {
    const double t = theta[i];
    if (t > sel[0] && t != 0.0) {
      lab[i] = (double)AIRG_C;
      conv = true;
    }
  }
  block_add(count, conv ? 1ull : 0ull);
}
// F points of this slab below global fine row `limit` (zero-diagonal message)
__global__ void k_f_below(int n, int64_t lo, const double* __restrict__ lab, unsigned long long limit,
                          unsigned long long* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool f = i < n && (unsigned long long)(lo + i) < limit && lab[i] == (double)AIRG_F;
  block_add(cnt, f ? 1ull : 0ull);
}

}  // namespace

// reverse exchange: every halo entry is added into its owner's slot
void reverse_add(Ctx& c, DHier& d, DVec& V) {
  const int P = V.part.P();
  if (d.me < 0) {
    for (int r = 0; r < P; ++r) {
      DVec::Rank& R = V.rk[r];
      if (R.nhalo)
        LAUNCH(c, k_scatter_add, blocks_for(R.nhalo, 256), 256, 0, R.nhalo, R.src_rank.p, R.src_idx.p,
               (double* const*)V.bases.p, (const double*)(R.buf.p + R.own));
    }
    return;
  }
  if (P == 1) return;
  DVec::Rank& M = V.rk[d.me];
  bool any = M.nhalo > 0;
  for (int q = 0; q < P && !any; ++q) any = M.send_cnt[q] || M.recv_cnt[q];
  if (!any) return;  // no traffic of mine in either direction
  NCCL_CHECK(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == d.me) continue;
    if (M.recv_cnt[q])
      NCCL_CHECK(ncclSend(M.buf.p + M.own + M.recv_off[q], (size_t)M.recv_cnt[q], ncclDouble, q, d.comm,
                          c.stream));
    if (M.send_cnt[q])
      NCCL_CHECK(ncclRecv(M.send_buf.p + M.send_off[q], (size_t)M.send_cnt[q], ncclDouble, q, d.comm,
                          c.stream));
  }
  NCCL_CHECK(ncclGroupEnd());
  const int64_t ns = M.send_off[P - 1] + M.send_cnt[P - 1];
  if (ns) LAUNCH(c, k_unpack_add, blocks_for(ns, 256), 256, 0, ns, M.send_idx.p, M.send_buf.p, M.buf.p);
}

void cf_split_slabs(Ctx& c, DHier& d, DVec& V, std::vector<Csr>& loc, double alpha, uint64_t seed,
                    bool ddc_enabled, double fraction, int64_t bins, std::vector<DBuf<double>>& labs,
                    CfReport& rep) {
  const int P = d.P, me = d.me;
  const ncclComm_t comm = d.comm;
  // Per rank: thr, |S_i|, w, theta (own rows); labels / marks travel in V's
  // [own | halo] buffers. Global counters: one shared block in emulation, one
  // per process + NCCL allreduces otherwise.
  // u: [0] |S| [1] n_f_pre [2] max theta bits [3] bad row [4] converted
  struct RS {
    DBuf<int32_t> s_cnt;
    DBuf<double> thr, w, lab, theta;
  };
  std::vector<RS> rs(P);
  auto mine = [&](auto&& f) {
    for (int r = 0; r < P; ++r)
      if (d.mine(r)) f(r);
  };
  const bool nccl = me >= 0 && P > 1;
  DBuf<unsigned long long> u(c, 8), hist(c, ddc_enabled ? (size_t)std::max<int64_t>(1, bins) : 1);
  DBuf<double> sel(c, 2);
  CUDA_CHECK(cudaMemsetAsync(u.p, 0, 8 * sizeof(unsigned long long), c.stream));
  CUDA_CHECK(cudaMemsetAsync(u.p + 3, 0xff, sizeof(unsigned long long), c.stream));
  hist.zero(c);
  sel.zero(c);
  auto allreduce = [&](unsigned long long* p, size_t cnt, ncclRedOp_t op) {
    if (nccl) NCCL_CHECK(ncclAllReduce(p, p, cnt, ncclUint64, op, comm, c.stream));
  };
  const uint64_t key = splitmix64_host(seed ^ splitmix64_host(0x57454947ull));
  // 1. thresholds, |S_i|, |S^T| contributions, then the reverse sum of the counts
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    R.buf.zero(c);
    const int n = (int)R.own;
    rs[r].s_cnt.alloc(c, (size_t)std::max(1, n));
    rs[r].thr.alloc(c, (size_t)std::max(1, n));
    if (n)
      LAUNCH(c, k_frows, blocks_for(n, 256), 256, 0, n, loc[r].rp.p, loc[r].ci.p, loc[r].v.p, alpha,
             rs[r].thr.p, rs[r].s_cnt.p, R.buf.p, u.p);
  });
  reverse_add(c, d, V);
  // 2. weights (own), forward exchange
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    const int n = (int)R.own;
    rs[r].w.alloc(c, (size_t)std::max<int64_t>(1, R.own + R.nhalo));
    if (n) LAUNCH(c, k_dweights, blocks_for(n, 256), 256, 0, n, R.lo, rs[r].s_cnt.p, R.buf.p, key, rs[r].w.p);
    if (n) CUDA_CHECK(cudaMemcpyAsync(R.buf.p, rs[r].w.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  });
  exchange(c, d, V);
  // 3. not-minimal marks from the strong entries (thresholds re-applied), reverse sum
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    const int64_t tot = R.own + R.nhalo;
    if (tot) CUDA_CHECK(cudaMemcpyAsync(rs[r].w.p, R.buf.p, sizeof(double) * tot, cudaMemcpyDeviceToDevice, c.stream));
    R.buf.zero(c);
    const int n = (int)R.own;
    if (n)
      LAUNCH(c, k_fmarks, blocks_for(n, 256), 256, 0, n, R.lo, R.own, R.halo.p, loc[r].rp.p, loc[r].ci.p,
             loc[r].v.p, rs[r].thr.p, rs[r].w.p, R.buf.p);
  });
  reverse_add(c, d, V);
  // 4. labels (own), n_f; forward exchange of the labels
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    const int n = (int)R.own;
    rs[r].lab.alloc(c, (size_t)std::max<int64_t>(1, R.own + R.nhalo));
    if (n) LAUNCH(c, k_flabels, blocks_for(n, 256), 256, 0, n, rs[r].w.p, R.buf.p, rs[r].lab.p, u.p + 1);
    if (n) CUDA_CHECK(cudaMemcpyAsync(R.buf.p, rs[r].lab.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  });
  allreduce(u.p, 2, ncclSum);
  exchange(c, d, V);
  if (ddc_enabled) {
    // 5. theta (own F rows) -> global max / bad row -> histogram -> alpha -> convert
    mine([&](int r) {
      DVec::Rank& R = V.rk[r];
      const int64_t tot = R.own + R.nhalo;
      if (tot) CUDA_CHECK(cudaMemcpyAsync(rs[r].lab.p, R.buf.p, sizeof(double) * tot, cudaMemcpyDeviceToDevice, c.stream));
      const int n = (int)R.own;
      rs[r].theta.alloc(c, (size_t)std::max(1, n));
      if (n)
        LAUNCH(c, k_ftheta, blocks_for(n, 256), 256, 0, n, R.lo, loc[r].rp.p, loc[r].ci.p, loc[r].v.p,
               rs[r].lab.p, rs[r].theta.p, u.p + 2, u.p + 3);
    });
    allreduce(u.p + 2, 1, ncclMax);
    allreduce(u.p + 3, 1, ncclMin);
    mine([&](int r) {
      const int n = (int)V.rk[r].own;
      const size_t smem = bins <= 8192 ? (size_t)bins * sizeof(unsigned) : 0;
      if (n)
        LAUNCH(c, k_fhist, (unsigned)std::min<int64_t>(blocks_for(n, 256), 4 * c.num_sms), 256, smem, n,
               rs[r].lab.p, rs[r].theta.p, u.p + 2, bins, hist.p);
    });
    allreduce(hist.p, (size_t)bins, ncclSum);
    launch_ddc_select(c, u.p + 1, hist.p, bins, fraction, u.p + 2, sel.p);
    mine([&](int r) {
      const int n = (int)V.rk[r].own;
      if (n) LAUNCH(c, k_fconvert, blocks_for(n, 256), 256, 0, n, rs[r].theta.p, sel.p, u.p + 3, rs[r].lab.p, u.p + 4);
    });
    allreduce(u.p + 4, 1, ncclSum);
  }
  unsigned long long hu[8];
  to_host(c, hu, u.p, 8);
  double hs[2];
  to_host(c, hs, sel.p, 2);
  if (ddc_enabled && hu[3] != ~0ull) {
    // the reference names the A_ff row: #F points before the global fine row
    DBuf<unsigned long long> cnt(c, 1);
    cnt.zero(c);
    mine([&](int r) {
      const int n = (int)V.rk[r].own;
      if (n) LAUNCH(c, k_f_below, blocks_for(n, 256), 256, 0, n, V.rk[r].lo, rs[r].lab.p, hu[3], cnt.p);
    });
    allreduce(cnt.p, 1, ncclSum);
    throw RuntimeError("dominance_report: zero diagonal in A_ff row " + std::to_string(read1(c, cnt.p)));
  }
  rep = CfReport();
  rep.s_nnz = (int64_t)hu[0];
  rep.n_f_pre = (int64_t)hu[1];
  rep.n_converted = (int64_t)hu[4];
  rep.n_f = rep.n_f_pre - rep.n_converted;
  rep.alpha_diag = hs[0];
  rep.max_theta = hs[1];
  // the converted labels of the halo (owners' final labels)
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    if (R.own) CUDA_CHECK(cudaMemcpyAsync(R.buf.p, rs[r].lab.p, sizeof(double) * R.own, cudaMemcpyDeviceToDevice, c.stream));
  });
  exchange(c, d, V);
  labs.resize(P);
  mine([&](int r) {
    DVec::Rank& R = V.rk[r];
    const int64_t tot = R.own + R.nhalo;
    if (tot) CUDA_CHECK(cudaMemcpyAsync(rs[r].lab.p, R.buf.p, sizeof(double) * tot, cudaMemcpyDeviceToDevice, c.stream));
    labs[r] = std::move(rs[r].lab);
  });
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

void dist_cf_split(Ctx& c, const Csr& a, int P, int me, ncclComm_t comm, const std::vector<int64_t>& starts,
                   double alpha, int64_t max_loops, uint64_t seed, bool ddc_enabled, double fraction,
                   int64_t bins, uint8_t* d_labels, CfReport& rep) {
  if (max_loops < 1) throw InvalidArgument("pmisr: max_loops must be >= 1");
  if (a.n != a.m) throw InvalidArgument("strength: matrix must be square");
  if ((int)starts.size() != P + 1 || starts[0] != 0 || starts[P] != a.n)
    throw InvalidArgument("dist: slab starts must cover the matrix");
  if (ddc_enabled && (fraction <= 0.0 || fraction > 1.0)) throw InvalidArgument("ddc: fraction must be in (0, 1]");
  if (P == 1) {  // one slab: no halo -- the fused one-GPU split (cfsplit.cu)
    const CfFused f = cf_split_fused(c, a, alpha, seed, ddc_enabled, fraction, bins, d_labels, nullptr);
    rep = CfReport();
    rep.s_nnz = f.s_nnz;
    rep.n_f_pre = f.n_f_pre;
    rep.n_converted = f.n_converted;
    rep.n_f = f.n_f_pre - f.n_converted;
    rep.max_theta = f.max_theta;
    rep.alpha_diag = f.alpha_diag;
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    return;
  }
  DHier d;
  d.P = P;
  d.me = me;
  d.comm = comm;
  DVec V;  // [own | halo] payloads: |S^T| counts, weights, marks, labels
  V.part.s = starts;
  V.N = a.n;
  V.rk.resize(P);
  std::vector<Csr> loc(P);
  for (int r = 0; r < P; ++r) {
    slice(c, a, V.part.lo(r), V.part.lo(r) + V.part.cnt(r), loc[r]);
    Marks mk;
    mk.init(c, a.n);
    mk.cols(c, loc[r], V.part.lo(r), V.part.lo(r) + V.part.cnt(r));
    set_halo(c, V, r, mk);
  }
  finalize(c, V, d);
  for (int r = 0; r < P; ++r)
    if (d.mine(r)) remap(c, loc[r], V, r);
  std::vector<DBuf<double>> labs;
  cf_split_slabs(c, d, V, loc, alpha, seed, ddc_enabled, fraction, bins, labs, rep);
  for (int r = 0; r < P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t n = V.rk[r].own, lo = me < 0 ? V.rk[r].lo : 0;
    if (n) LAUNCH(c, k_to_u8, blocks_for(n, 256), 256, 0, n, labs[r].p, d_labels + lo);
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// ---------------------------------------------------------------------------
void halo_plan_host(const std::vector<int64_t>& starts, int rank, const int64_t* cols, int64_t ncols,
                    std::vector<int64_t>& halo, std::vector<int64_t>& recv_cnt) {
  Part p;
  p.s = starts;
  const int64_t lo = p.lo(rank), hi = lo + p.cnt(rank);
  halo.clear();
  for (int64_t k = 0; k < ncols; ++k) {
    const int64_t g = cols[k] & 0x7fffffffLL;
    if (g < lo || g >= hi) halo.push_back(g);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  recv_cnt.assign(p.P(), 0);
  for (int64_t g : halo) recv_cnt[p.owner(g)]++;
}

void dist_create(Ctx& c, Hier& h, int P, int me, ncclComm_t comm, double threshold,
                 const int64_t* level0_starts, DHier& d) {
  if (P < 1) throw InvalidArgument("dist: need at least one rank");
  if (me >= P) throw InvalidArgument("dist: rank out of range");
  if (me >= 0 && P > 1 && !comm) throw InvalidArgument("dist: a communicator is needed per rank");
  d.P = P;
  d.me = me;
  d.comm = comm;
  d.threshold = threshold;
  const int L = (int)h.levels.size();
  d.top_n = h.top_n();
  // ---- partitions: the reference replay rule, then the coarse gather
  d.lv.resize(L);
  int active = P;
  // AIRG_DIST_MIN_ROWS (default 0 = off): beside the reference's locality
  // rule, halve the active ranks while a level has fewer rows per active rank
  // than this. Over NVLink the halo bytes of the slab partitions are
  // negligible (tools/dist_model.py: < 30 MB per V-cycle at 8 ranks, ~4 us
  // of link time) while every exchange costs a latency; below ~10^5 rows per
  // rank the row kernels sit at their launch floor, so fewer, fuller ranks
  // remove exchanges without adding kernel time. Any partition gives the
  // same bits.
  const int64_t min_rows = [] {
    const char* e = getenv("AIRG_DIST_MIN_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    const Csr& A = h.levels[l].a;
    Part p = (l == 0 && level0_starts) ? Part{std::vector<int64_t>(level0_starts, level0_starts + P + 1)}
                                       : balanced(A.n, active, P);
    D.ratio_before = locality(c, A, p, &D.share_before);
    D.ratio_after = D.ratio_before;
    D.share_after = D.share_before;
    // A caller-fixed level-0 partition (one process per GPU: the caller's b
    // and x slabs) is kept as given; halving applies from level 1 onward.
    const bool fixed = l == 0 && level0_starts;
    if (!fixed && D.ratio_before < threshold && active > 1) {
      const int na = (active + 1) / 2;
      p = merged(p, active, na);
      active = na;
      D.triggered = true;
      D.ratio_after = locality(c, A, p, &D.share_after);
    }
    while (!fixed && min_rows > 0 && active > 1 && (int64_t)A.n < min_rows * (int64_t)active) {
      const int na = (active + 1) / 2;
      p = merged(p, active, na);
      active = na;
      D.triggered = true;
      D.ratio_after = locality(c, A, p, &D.share_after);
    }
    D.active = active;
    D.fine = p;
  }
  // ---- pieces: every rank's slices of the global hierarchy
  DistPieces pc;
  pc.all_ranks = true;
  pc.coarse_n = h.coarse_a.n;
  pc.lv.resize(L);
  pc.fpart.resize(L);
  pc.n.resize(L);
  pc.nf.resize(L);
  for (int l = 0; l < L; ++l) {
    const DLevel& D = d.lv[l];
    const Level& Lv = h.levels[l];
    pc.n[l] = Lv.a.n;
    pc.nf[l] = Lv.map.nf;
    // F partition: #F points below each fine boundary
    DBuf<int64_t> bnd(c, (size_t)P + 1), cnt(c, (size_t)P + 1);
    to_device(c, bnd.p, D.fine.s.data(), (size_t)P + 1);
    LAUNCH(c, k_count_below, 1, 64, 0, Lv.map.f_to_fine.p, (int64_t)Lv.map.nf, bnd.p, P + 1, cnt.p);
    pc.fpart[l].s.resize(P + 1);
    to_host(c, pc.fpart[l].s.data(), cnt.p, (size_t)P + 1);
  }
  const Part cpart = gathered(h.coarse_a.n, P);
  pc.fused_smooths = h.fused_smooths;
  if (h.fused_smooths >= 0)
    for (int l = 0; l < L; ++l) {
      d.lv[l].nnz_afp = h.levels[l].afp.nnz;
      d.lv[l].nnz_w = h.levels[l].fw.nnz;
    }
  pc.AC.resize(P);
  pc.ACI.resize(P);
  pc.A0.resize(P);
  for (int l = 0; l < L; ++l) {
    const Level& Lv = h.levels[l];
    const Part& coarse = l + 1 < L ? d.lv[l + 1].fine : cpart;
    pc.lv[l].resize(P);
    for (int r = 0; r < P; ++r) {
      DistPieces::LevelRank& R = pc.lv[l][r];
      const int64_t flo = pc.fpart[l].lo(r), fhi = flo + pc.fpart[l].cnt(r);
      const int64_t clo = coarse.lo(r), chi = clo + coarse.cnt(r);
      const int64_t lo = d.lv[l].fine.lo(r), hi = lo + d.lv[l].fine.cnt(r);
      slice(c, Lv.r, clo, chi, R.R);
      slice(c, Lv.af, flo, fhi, R.AF);
      slice(c, Lv.affg, flo, fhi, R.AFFG);
      slice(c, Lv.ffinv, flo, fhi, R.FINV);
      if (h.fused_smooths >= 0) {  // the fast V-cycle's fused operators, by F rows
        slice(c, Lv.afp, flo, fhi, R.AFP);
        slice(c, Lv.fw, flo, fhi, R.W);
      }
      R.pmap.alloc(c, (size_t)std::max<int64_t>(1, hi - lo));
      if (hi > lo)
        CUDA_CHECK(cudaMemcpyAsync(R.pmap.p, Lv.pmap.p + lo, sizeof(int32_t) * (hi - lo),
                                   cudaMemcpyDeviceToDevice, c.stream));
      R.f2f.alloc(c, (size_t)std::max<int64_t>(1, fhi - flo));
      if (fhi > flo)
        CUDA_CHECK(cudaMemcpyAsync(R.f2f.p, Lv.map.f_to_fine.p + flo, sizeof(int32_t) * (fhi - flo),
                                   cudaMemcpyDeviceToDevice, c.stream));
    }
  }
  const Part& top = L ? d.lv[0].fine : cpart;
  for (int r = 0; r < P; ++r) {
    slice(c, h.coarse_a, cpart.lo(r), cpart.lo(r) + cpart.cnt(r), pc.AC[r]);
    slice(c, h.coarse_inv, cpart.lo(r), cpart.lo(r) + cpart.cnt(r), pc.ACI[r]);
    const Csr& A0 = L ? h.levels[0].a : h.coarse_a;
    slice(c, A0, top.lo(r), top.lo(r) + top.cnt(r), pc.A0[r]);
  }
  dist_build(c, d, pc);
}

void dist_build(Ctx& c, DHier& d, DistPieces& pc) {
  const int P = d.P;
  const int L = (int)d.lv.size();
  auto have = [&](int r) { return pc.all_ranks || d.mine(r); };
  d.cpart = gathered(pc.coarse_n, P);
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    D.coarse_part = l + 1 < L ? d.lv[l + 1].fine : d.cpart;
    D.fpart = pc.fpart[l];
    D.rk.resize(P);
    D.B.part = D.fine;
    D.B.N = pc.n[l];
    D.X.part = D.fine;
    D.X.N = pc.n[l];
    D.RF.part = D.fpart;
    D.RF.N = pc.nf[l];
    D.B.rk.resize(P);
    D.X.rk.resize(P);
    D.RF.rk.resize(P);
  }
  d.CB.part = d.cpart;
  d.CX.part = d.cpart;
  d.CR.part = d.cpart;
  d.CB.N = d.CX.N = d.CR.N = pc.coarse_n;
  d.CB.rk.resize(P);
  d.CX.rk.resize(P);
  d.CR.rk.resize(P);
  d.XS.part = L ? d.lv[0].fine : d.cpart;
  d.XS.N = L ? pc.n[0] : pc.coarse_n;
  d.XS.rk.resize(P);
  d.rk.resize(P);

  // ---- the ranks' operators (global columns) and their halos (all ranks
  // when every piece is here: the peers' halo lists give the send lists)
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    for (int r = 0; r < P; ++r) {
      if (!have(r)) continue;
      DLevel::Rank& R = D.rk[r];
      DistPieces::LevelRank& S = pc.lv[l][r];
      const int64_t flo = D.fpart.lo(r), fhi = flo + D.fpart.cnt(r);
      const int64_t lo = D.fine.lo(r), hi = lo + D.fine.cnt(r);
      R.R = std::move(S.R);
      R.AF = std::move(S.AF);
      R.AFFG = std::move(S.AFFG);
      R.FINV = std::move(S.FINV);
      if (pc.fused_smooths >= 0) {
        R.AFP = std::move(S.AFP);
        R.W = std::move(S.W);
      }
      if (pc.fused_smooths >= 0 && d.mine(r)) {  // own C rows (the complement of the F rows)
        std::vector<int32_t> fh((size_t)(fhi - flo));
        if (fhi > flo) to_host(c, fh.data(), S.f2f.p, fh.size());
        std::vector<char> isf((size_t)(hi - lo), 0);
        for (int32_t g : fh) isf[(size_t)(g - lo)] = 1;
        std::vector<int32_t> ch;
        ch.reserve((size_t)(hi - lo - (fhi - flo)));
        for (int64_t i = 0; i < hi - lo; ++i)
          if (!isf[(size_t)i]) ch.push_back((int32_t)i);
        R.nc_own = (int64_t)ch.size();
        R.c2f.alloc(c, std::max<size_t>(1, ch.size()));
        if (!ch.empty()) to_device(c, R.c2f.p, ch.data(), ch.size());
      }
      R.nf_own = fhi - flo;
      R.n_own = hi - lo;
      R.pmap = std::move(S.pmap);
      R.f2f.alloc(c, (size_t)std::max<int64_t>(1, fhi - flo));
      if (fhi > flo) LAUNCH(c, k_shift, blocks_for(fhi - flo, 256), 256, 0, fhi - flo, S.f2f.p, lo, R.f2f.p);
      R.sc.alloc(c, (size_t)std::max<int64_t>(1, fhi - flo));
      // halos: B_l <- R_l ; X_l <- AF, AFFG, P_{l-1} ; RF_l <- FINV
      Marks mb, mx, mf;
      mb.init(c, D.B.N);
      mb.cols(c, R.R, lo, hi);
      set_halo(c, D.B, r, mb);
      mx.init(c, D.X.N);
      mx.cols(c, R.AF, lo, hi);
      mx.cols(c, R.AFFG, lo, hi);
      if (l > 0) {
        const DLevel::Rank& U = d.lv[l - 1].rk[r];
        mx.vals(c, U.pmap.p, U.n_own, lo, hi);
        if (pc.fused_smooths >= 0 && U.AFP.n) mx.cols(c, U.AFP, lo, hi);  // the coarser level's A_F P reads X_l
      }
      set_halo(c, D.X, r, mx);
      mf.init(c, D.RF.N);
      mf.cols(c, R.FINV, flo, fhi);
      if (pc.fused_smooths >= 0 && R.W.n) mf.cols(c, R.W, flo, fhi);
      set_halo(c, D.RF, r, mf);
    }
  }
  // coarsest: A_c / Ac^-1 on their owner, CX halo also serves P_{L-1}
  for (int r = 0; r < P; ++r) {
    if (!have(r)) continue;
    DHier::Rank& T = d.rk[r];
    const int64_t lo = d.cpart.lo(r), hi = lo + d.cpart.cnt(r);
    T.AC = std::move(pc.AC[r]);
    T.ACI = std::move(pc.ACI[r]);
    Marks mc, mb, mr;
    mc.init(c, d.CX.N);
    mc.cols(c, T.AC, lo, hi);
    if (L) {
      const DLevel::Rank& U = d.lv[L - 1].rk[r];
      mc.vals(c, U.pmap.p, U.n_own, lo, hi);
      if (pc.fused_smooths >= 0 && U.AFP.n) mc.cols(c, U.AFP, lo, hi);
    }
    set_halo(c, d.CX, r, mc);
    mb.init(c, d.CB.N);
    mb.cols(c, T.ACI, lo, hi);
    set_halo(c, d.CB, r, mb);
    mr.init(c, d.CR.N);
    mr.cols(c, T.ACI, lo, hi);
    set_halo(c, d.CR, r, mr);
    // top operator for the residual
    const int64_t tlo = d.XS.part.lo(r), thi = tlo + d.XS.part.cnt(r);
    T.A0 = std::move(pc.A0[r]);
    Marks ms;
    ms.init(c, d.XS.N);
    ms.cols(c, T.A0, tlo, thi);
    set_halo(c, d.XS, r, ms);
    T.rhs.alloc(c, (size_t)std::max<int64_t>(1, thi - tlo));
  }
  // ---- buffers, tables, remapped columns
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    finalize(c, D.B, d, pc.all_ranks);
    finalize(c, D.X, d, pc.all_ranks);
    finalize(c, D.RF, d, pc.all_ranks);
  }
  finalize(c, d.CB, d, pc.all_ranks);
  finalize(c, d.CX, d, pc.all_ranks);
  finalize(c, d.CR, d, pc.all_ranks);
  finalize(c, d.XS, d, pc.all_ranks);
  if (p2p_requested() && P > 1) {  // the solve's exchanged vectors move to the p2p arenas
    std::vector<DVec*> vecs;
    for (int l = 0; l < L; ++l) {
      vecs.push_back(&d.lv[l].B);
      vecs.push_back(&d.lv[l].X);
      vecs.push_back(&d.lv[l].RF);
    }
    vecs.push_back(&d.CX);
    vecs.push_back(&d.CR);
    vecs.push_back(&d.XS);
    p2p_setup(c, d, vecs);
  }
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    const DVec& Xn = l + 1 < L ? d.lv[l + 1].X : d.CX;
    for (int r = 0; r < P; ++r) {
      DLevel::Rank& R = D.rk[r];
      if (!d.mine(r)) {
        R = DLevel::Rank();
        continue;
      }
      remap(c, R.R, D.B, r);
      remap(c, R.AF, D.X, r);
      remap(c, R.AFFG, D.X, r);
      remap(c, R.FINV, D.RF, r);
      if (pc.fused_smooths >= 0) {
        remap(c, R.AFP, Xn, r);
        remap(c, R.W, D.RF, r);
      }
      const DVec::Rank& XR = Xn.rk[r];
      if (R.n_own)
        LAUNCH(c, k_remap_vals, blocks_for(R.n_own, 256), 256, 0, R.n_own, R.pmap.p, R.pmap.p, XR.lo,
               XR.lo + XR.own, XR.own, XR.halo.p, XR.nhalo);
    }
  }
  d.nparts = 0;
  d.part_off.assign(P, 0);
  for (int r = 0; r < P; ++r) {
    DHier::Rank& T = d.rk[r];
    if (!d.mine(r)) {
      T = DHier::Rank();
      continue;
    }
    remap(c, T.AC, d.CX, r);
    remap(c, T.ACI, d.CR, r);  // CB and CR share the column space; CR's halo is used
    remap(c, T.A0, d.XS, r);
    d.part_off[r] = d.nparts;
    d.nparts += (int)blocks_for(std::max(1, T.A0.n), kTileThreads);
  }
  d.part.alloc(c, (size_t)d.nparts + 8);
  d.scal.alloc(c, 8);
  d.fused_smooths = pc.fused_smooths;
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

namespace {

bool dist_fast(const DHier& d, const airg_solve_config& cfg) {
  return cfg.fast != 0 && d.fused_smooths >= 0 && d.fused_smooths == cfg.up_f_smooths;
}

// the composed coarse solve for the fast V-cycle (on the coarse grid's
// owner; every rank agrees on whether it is used)
void dist_coarse_compose(Ctx& c, DHier& d, const airg_solve_config& cfg) {
  if (!dist_fast(d, cfg) || d.coarse_e_its == cfg.coarse_iterations) return;
  int ok = 1;
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    DHier::Rank& T = d.rk[r];
    T.ACE = Csr();
    if (T.AC.n && !compose_coarse(c, T.AC, T.ACI, cfg.coarse_iterations, T.ACE)) ok = 0;
  }
  if (d.me >= 0 && d.P > 1) {  // the coarse owner's answer to every rank
    DBuf<int> f(c, 1);
    to_device(c, f.p, &ok, 1);
    NCCL_CHECK(ncclAllReduce(f.p, f.p, 1, ncclInt, ncclMin, d.comm, c.stream));
    to_host(c, &ok, f.p, 1);
  }
  for (int r = 0; r < d.P; ++r)
    if (d.mine(r) && d.rk[r].ACE.n) row_max(c, {&d.rk[r].ACE});
  d.coarse_e_ok = ok != 0;
  d.coarse_e_its = cfg.coarse_iterations;
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

void enqueue_vcycle(Ctx& c, DHier& d, const airg_solve_config& cfg) {
  const int L = (int)d.lv.size();
  const int P = d.P;
  // fast mode (the single-GPU fast V-cycle's fused level operators on the
  // slabs, lane-group row kernels): per level R b on the way down; on the way
  // up x = P e_c, r1 = b_F - (A_F P) e_c, x_F += W_k r1 -- three passes
  // instead of 1 + 2 k, same halos plus A_F P's coarse and W's F columns
  const bool fast = dist_fast(d, cfg);
  auto rank_loop = [&](auto&& f) {
    for (int r = 0; r < P; ++r)
      if (d.mine(r)) f(r);
  };
  // descent
  for (int l = 0; l < L; ++l) {
    DLevel& D = d.lv[l];
    exchange(c, d, D.B);
    DVec& Bn = l + 1 < L ? d.lv[l + 1].B : d.CB;
    rank_loop([&](int r) {
      const Csr& R = D.rk[r].R;
      if (R.n)
        launch_rows(c, R, (const double*)D.B.rk[r].buf.p, LStore{Bn.rk[r].buf.p}, fast);
    });
    release(c, d, D.B);
  }
  // coarse solve on the coarse owner(s); CB and CR feed Ac^-1 through CR's
  // layout: copy the owned rhs into CR before the first application. Fast
  // mode with the composed E_k (the coarse grid is gathered: no halo): e = E_k b.
  if (fast && d.coarse_e_ok && d.coarse_e_its == cfg.coarse_iterations) {
    rank_loop([&](int r) {
      const Csr& E = d.rk[r].ACE;
      if (E.n) launch_rows(c, E, (const double*)d.CB.rk[r].buf.p, LStore{d.CX.rk[r].buf.p}, true);
    });
  }
  for (int64_t it = 0; !(fast && d.coarse_e_ok && d.coarse_e_its == cfg.coarse_iterations) &&
                       it < cfg.coarse_iterations; ++it) {
    if (it == 0) {
      rank_loop([&](int r) {
        const int64_t own = d.CB.rk[r].own;
        if (own)
          CUDA_CHECK(cudaMemcpyAsync(d.CR.rk[r].buf.p, d.CB.rk[r].buf.p, sizeof(double) * own,
                                     cudaMemcpyDeviceToDevice, c.stream));
      });
    } else {
      exchange(c, d, d.CX);
      rank_loop([&](int r) {
        const Csr& A = d.rk[r].AC;
        if (A.n)
          launch_rows(c, A, (const double*)d.CX.rk[r].buf.p, LCres{d.CB.rk[r].buf.p, d.CR.rk[r].buf.p});
      });
      release(c, d, d.CX);
    }
    exchange(c, d, d.CR);
    rank_loop([&](int r) {
      const Csr& A = d.rk[r].ACI;
      if (A.n)
        launch_rows(c, A, (const double*)d.CR.rk[r].buf.p, LCupd{d.CX.rk[r].buf.p, it == 0 ? 1 : 0});
    });
    release(c, d, d.CR);
  }
  // ascent
  for (int l = L - 1; fast && l >= 0; --l) {
    DLevel& D = d.lv[l];
    DVec& Xn = l + 1 < L ? d.lv[l + 1].X : d.CX;
    const bool smooth = cfg.up_f_smooths > 0;
    exchange(c, d, Xn);
    if (smooth) {
      rank_loop([&](int r) {
        const DLevel::Rank& R = D.rk[r];
        if (R.nf_own)
          launch_rows(c, R.AFP, (const double*)Xn.rk[r].buf.p,
                      LFres1P{D.B.rk[r].buf.p, R.f2f.p, D.RF.rk[r].buf.p}, true);
      });
      exchange(c, d, D.RF);
    }
    // x_l = P e_c + [W r1 on the F rows] in one pass (fusedx.cuh)
    rank_loop([&](int r) {
      const DLevel::Rank& R = D.rk[r];
      if (R.n_own)
        launch_fused_x_raw(c, R.W, D.RF.rk[r].buf.p, R.f2f.p, R.c2f.p, (int)R.nc_own, R.pmap.p, Xn.rk[r].buf.p,
                           D.X.rk[r].buf.p, false, smooth);
    });
    if (smooth) release(c, d, D.RF);
    release(c, d, Xn);
  }
  for (int l = L - 1; !fast && l >= 0; --l) {
    DLevel& D = d.lv[l];
    DVec& Xn = l + 1 < L ? d.lv[l + 1].X : d.CX;
    exchange(c, d, Xn);
    rank_loop([&](int r) {
      const DLevel::Rank& R = D.rk[r];
      if (R.n_own)
        LAUNCH_PDL(c, k_prolong4_l, blocks_for(R.n_own / 4 + 1, 256), 256, 0, (int)R.n_own, R.pmap.p,
                   Xn.rk[r].buf.p, D.X.rk[r].buf.p);
    });
    release(c, d, Xn);
    for (int64_t s = 0; s < cfg.up_f_smooths; ++s) {
      exchange(c, d, D.X);
      rank_loop([&](int r) {
        DLevel::Rank& R = D.rk[r];
        if (!R.nf_own) return;
        const double* bl = D.B.rk[r].buf.p;
        if (s == 0)
          launch_rows_fc(c, R.AF, (const double*)D.X.rk[r].buf.p, LFres1{bl, R.f2f.p, D.RF.rk[r].buf.p, R.sc.p});
        else
          launch_rows(c, R.AFFG, (const double*)D.X.rk[r].buf.p, LFres2{bl, R.f2f.p, R.sc.p, D.RF.rk[r].buf.p});
      });
      release(c, d, D.X);
      exchange(c, d, D.RF);
      rank_loop([&](int r) {
        DLevel::Rank& R = D.rk[r];
        if (!R.nf_own) return;
        launch_rows(c, R.FINV, (const double*)D.RF.rk[r].buf.p, LFupd{R.f2f.p, D.X.rk[r].buf.p});
      });
      release(c, d, D.RF);
    }
  }
}

// x += e (owned), r = b - A x, ||r||^2 -> d.scal[0] (local sum under NCCL)
void enqueue_update_residual(Ctx& c, DHier& d) {
  const int L = (int)d.lv.size();
  DVec& E = L ? d.lv[0].X : d.CX;
  DVec& Rv = L ? d.lv[0].B : d.CB;
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t own = d.XS.rk[r].own;
    if (own)
      LAUNCH_PDL(c, k_axpy1_l, blocks_for(own / 2 + 1, 256), 256, 0, (int)own, (const double*)E.rk[r].buf.p,
                 d.XS.rk[r].buf.p);
  }
  exchange(c, d, d.XS);
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    const Csr& A = d.rk[r].A0;
    if (A.n)
      launch_rows(c, A, (const double*)d.XS.rk[r].buf.p,
                  LResid{d.rk[r].rhs.p, Rv.rk[r].buf.p, d.part.p + d.part_off[r], 0.0});
    else
      CUDA_CHECK(cudaMemsetAsync(d.part.p + d.part_off[r], 0, sizeof(double), c.stream));
  }
  release(c, d, d.XS);
  p2p_flush(c, d);  // the captured body hands back every slot it read
  LAUNCH_PDL(c, k_sum, 1, 1024, 0, (const double*)d.part.p, d.nparts, d.scal.p);
}

double read_norm2(Ctx& c, DHier& d, double* dev) {
  if (d.me >= 0 && d.P > 1)
    NCCL_CHECK(ncclAllReduce(dev, dev, 1, ncclDouble, ncclSum, d.comm, c.stream));
  return read1(c, dev);
}

template <class F>
uint64_t capture_graph(Ctx& c, cudaGraphExec_t* exec, F&& body) {
  if (*exec) {
    cudaGraphExecDestroy(*exec);
    *exec = nullptr;
  }
  const uint64_t before = c.launches;
  cudaGraph_t g;
  CUDA_CHECK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(c.stream, &dummy);
    if (dummy) cudaGraphDestroy(dummy);
    throw;
  }
  CUDA_CHECK(cudaStreamEndCapture(c.stream, &g));
  CUDA_CHECK(cudaGraphInstantiate(exec, g, 0));
  CUDA_CHECK(cudaGraphDestroy(g));
  const uint64_t k = c.launches - before;
  c.launches = before;
  return k;
}

}  // namespace

namespace {

// ---- outer GMRES over the row slabs ------------------------------------------
// Local pieces of the single-GPU method (solve.cu gmres): per-rank partial
// dots of w with V_0..V_j (grid: blocks x (j+1)), summed over the blocks in
// a fixed order, then over the ranks (rank order in emulation, NCCL
// allreduce with one rank per GPU).
constexpr int kGmDotBlocks = 64;
__global__ void k_gmd_dots(int64_t n, const double* __restrict__ V, const double* __restrict__ w,
                           double* __restrict__ part) {
  __shared__ double sm[32];
  const double* vk = V + (int64_t)blockIdx.y * n;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(vk[i], w[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void k_gmd_fold(const double* __restrict__ part, int np, double* __restrict__ out) {
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int b = 0; b < np; ++b) s += part[(int64_t)blockIdx.x * np + b];
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}
// w -= V(:, 0..j) h
__global__ void k_gmd_update(int64_t n, int jp1, const double* __restrict__ V, const double* __restrict__ h,
                             double* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = w[i];
  for (int k = 0; k < jp1; ++k) s -= h[k] * V[(int64_t)k * n + i];
  w[i] = s;
}
// dst = src * a (and dst2 = the same)
__global__ void k_gmd_scale(int64_t n, const double* __restrict__ src, double a, double* __restrict__ dst,
                            double* __restrict__ dst2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = a == 0.0 ? 0.0 : src[i] * a;
  dst[i] = v;
  if (dst2) dst2[i] = v;
}
// x += Z(:, 0..j-1) y
__global__ void k_gmd_xupdate(int64_t n, int j, const double* __restrict__ Z, const double* __restrict__ y,
                              double* __restrict__ x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = x[i];
  for (int k = 0; k < j; ++k) s += y[k] * Z[(int64_t)k * n + i];
  x[i] = s;
}

}  // namespace

// Right-preconditioned restarted GMRES around the distributed V-cycle (the
// steps of the single-GPU gmres(), solve.cu, and of the serial restatement,
// oracle/airg_oracle.c): rows, vectors and Krylov basis are row slabs of
// level 0; every inner product is a local partial followed by one
// allreduce of (j + 1) values; the Hessenberg least squares runs on the host.
namespace {
// emulation: every rank's copy of cnt doubles <- their sum in rank order
__global__ void k_rank_allsum(int P, int cnt, double* const* __restrict__ p) {
  pdl_wait();
  pdl_trigger();
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += p[q][k];
    for (int q = 0; q < P; ++q) p[q][k] = s;
  }
}
// sum of np partials (one block, fixed tree)
__global__ void k_sum_part(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double sm[32];
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
  }
}
}  // namespace

// Device-resident distributed GMRES(m): the one-GPU device GMRES's kernels
// (gmres.cuh: Gram-corrected CGS2 over the unnormalised basis, Givens and
// the stopping tests on the device) on every rank's slab, the three
// reductions of a step (the dots with the Gram column, the norm, and per
// restart the residual norm) summed over the ranks by an NCCL allreduce
// (emulation: one kernel in rank order), so every rank holds the same
// scalars. No host round trip inside a restart cycle: the host stays one
// Arnoldi step ahead and reads the lagged "continue" flag of the previous
// step (a step enqueued past the end is a no-op in k_gm_step).
void dist_gmres_dev(Ctx& c, DHier& d, const airg_solve_config& cfg, const double* d_b, double* d_x,
                    airg_solve_stats& st, std::vector<double>& hist) {
  const int L = (int)d.lv.size();
  const int P = d.P;
  const int m = (int)(cfg.gmres_restart > 0 ? cfg.gmres_restart : 30);
  const bool fast = dist_fast(d, cfg);
  DVec& In = L ? d.lv[0].B : d.CB;
  DVec& Out = L ? d.lv[0].X : d.CX;
  auto own = [&](int r) { return d.XS.rk[r].own; };
  const int64_t cap = std::max<int64_t>(2, cfg.max_iterations + 2);
  const int rq = d.me < 0 ? 0 : d.me;  // the rank whose (identical) state the host reads
  if (d.gm_m != m || (int)d.gm.size() != P || !d.gm[rq].st.p || d.gm[rq].hist.n < (size_t)cap) {
    d.gm.clear();
    d.gm.resize(P);
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      const size_t o = (size_t)std::max<int64_t>(1, own(r));
      DHier::GmRank& G = d.gm[r];
      // one column beyond V_0..V_m and Z_0..Z_{m-1}: the step enqueued past
      // the end of a cycle (a no-op for the scalars) still writes V_{j+1}, Z_j
      G.V.alloc(c, o * (m + 2));
      G.Z.alloc(c, o * (m + 1));
      G.w.alloc(c, o);
      G.x.alloc(c, o);
      G.st.alloc(c, 1);
      G.H.alloc(c, (size_t)(kGmMax + 1) * kGmMax);
      G.cs.alloc(c, kGmMax);
      G.sn.alloc(c, kGmMax);
      G.g.alloc(c, kGmMax + 1);
      G.y.alloc(c, kGmMax);
      G.hb.alloc(c, 7 * (kGmMax + 1));
      G.G.alloc(c, (size_t)(kGmMax + 1) * (kGmMax + 1));
      G.hist.alloc(c, (size_t)cap);
      G.gpart.alloc(c, (size_t)2 * (kGmMax + 1) * (size_t)std::max(1, gm_blocks(own(r))));
      G.sc.alloc(c, 2);
    }
    d.gm_m = m;
  }
  if (!d.gm_flag) CUDA_CHECK(cudaMallocHost(&d.gm_flag, 2 * sizeof(int)));
  dist_coarse_compose(c, d, cfg);
  const int64_t vkey = (cfg.up_f_smooths * 1000003 + cfg.coarse_iterations * 31) * 2 + (fast ? 1 : 0);
  if (!d.graph_vc || d.graph_vc_key != vkey) {
    d.graph_vc_kernels = capture_graph(c, &d.graph_vc, [&] {
      enqueue_vcycle(c, d, cfg);
      p2p_flush(c, d);
    });
    d.graph_vc_key = vkey;
  }
  auto mine = [&](auto&& f) {
    for (int r = 0; r < P; ++r)
      if (d.mine(r)) f(r);
  };
  // segments of hb: (h1) | h2 | nrm | d (2 (kGmMax + 1)) | hsum | vs
  const int S = kGmMax + 1;
  auto h2 = [&](int r) { return d.gm[r].hb.p + S; };
  auto nrm = [&](int r) { return d.gm[r].hb.p + 2 * S; };
  auto dd = [&](int r) { return d.gm[r].hb.p + 3 * S; };
  auto hsum = [&](int r) { return d.gm[r].hb.p + 5 * S; };
  auto vs = [&](int r) { return d.gm[r].hb.p + 6 * S; };
  // allreduce sites: pointer tables for the emulated reduction
  DBuf<double*> pd(c, (size_t)P), pn(c, (size_t)P), ps(c, (size_t)P);
  if (d.me < 0 && P > 1) {
    std::vector<double*> a(P), b(P), e(P);
    for (int r = 0; r < P; ++r) {
      a[r] = dd(r);
      b[r] = nrm(r);
      e[r] = d.gm[r].sc.p;
    }
    to_device(c, pd.p, a.data(), (size_t)P);
    to_device(c, pn.p, b.data(), (size_t)P);
    to_device(c, ps.p, e.data(), (size_t)P);
  }
  auto allsum = [&](int cnt, double* const* table, const std::function<double*(int)>& mineptr) {
    if (P == 1) return;
    if (d.me >= 0) {
      double* p = mineptr(d.me);
      NCCL_CHECK(ncclAllReduce(p, p, (size_t)cnt, ncclDouble, ncclSum, d.comm, c.stream));
    } else {
      LAUNCH_PDL(c, k_rank_allsum, 1, 256, 0, P, cnt, table);
    }
  };
  // w (or x for the residual) -> A x over the slabs, epilogue per rank
  auto stage_xs = [&](const std::function<const double*(int)>& xin) {
    mine([&](int r) {
      if (own(r))
        CUDA_CHECK(cudaMemcpyAsync(d.XS.rk[r].buf.p, xin(r), sizeof(double) * own(r), cudaMemcpyDeviceToDevice,
                                   c.stream));
    });
    exchange(c, d, d.XS);
  };
  // ---- start: r = b, x = 0, ||b||
  GmDev s0 = {};
  s0.cap = cap;
  s0.maxit = cfg.max_iterations;
  s0.m = m;
  s0.rtol = cfg.rtol;
  mine([&](int r) {
    const int64_t o = own(r), lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    if (o) {
      CUDA_CHECK(cudaMemcpyAsync(d.rk[r].rhs.p, d_b + lo, sizeof(double) * o, cudaMemcpyDeviceToDevice, c.stream));
      CUDA_CHECK(cudaMemcpyAsync(d.gm[r].w.p, d_b + lo, sizeof(double) * o, cudaMemcpyDeviceToDevice, c.stream));
      dot_async(c, d.gm[r].w.p, d.gm[r].w.p, o, d.gm[r].sc.p, d.gm[r].gpart.p);
    } else {
      CUDA_CHECK(cudaMemsetAsync(d.gm[r].sc.p, 0, sizeof(double), c.stream));
    }
    CUDA_CHECK(cudaMemsetAsync(d.gm[r].x.p, 0, sizeof(double) * std::max<int64_t>(1, o), c.stream));
    to_device(c, d.gm[r].st.p, &s0, 1);
  });
  allsum(1, ps.p, [&](int r) { return d.gm[r].sc.p; });
  mine([&](int r) { LAUNCH(c, k_gm_init, 1, 32, 0, 0, 0, (const double*)d.gm[r].sc.p, d.gm[r].st.p, d.gm[r].hist.p); });
  GmDev s1;
  to_host(c, &s1, d.gm[rq].st.p, 1);
  bool outer = s1.bnorm != 0.0 && s1.maxit > 0;
  cudaEvent_t ev[2];
  CUDA_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const uint64_t l0 = c.launches;
  while (outer) {
    mine([&](int r) {
      LAUNCH(c, k_gm_cycle, (unsigned)gm_blocks(std::max<int64_t>(1, own(r))), kGmThreads, 0, 0, 0, own(r),
             (const double*)d.gm[r].w.p, d.gm[r].st.p, d.gm[r].V.p, In.rk[r].buf.p, d.gm[r].g.p, vs(r));
    });
    for (int k = 0;; ++k) {
      // ---- one Arnoldi step
      CUDA_CHECK(cudaGraphLaunch(d.graph_vc, c.stream));
      c.launches += d.graph_vc_kernels;
      stage_xs([&](int r) { return (const double*)Out.rk[r].buf.p; });
      mine([&](int r) {
        const Csr& A = d.rk[r].A0;
        if (A.n)
          launch_rows(c, A, (const double*)d.XS.rk[r].buf.p,
                      EpiGmSpmv{d.gm[r].w.p, Out.rk[r].buf.p, d.gm[r].Z.p, d.gm[r].st.p, own(r), vs(r)}, fast);
      });
      release(c, d, d.XS);
      p2p_flush(c, d);
      std::vector<int> nsf(P, 1);
      mine([&](int r) {
        const int64_t n = own(r);
        const int pp = n % 4 == 0 ? 2 : (n % 2 == 0 ? 1 : 0);
        double* part = d.gm[r].gpart.p;
        const double* V = d.gm[r].V.p;
        if (pp) {
          nsf[r] = (int)std::max<int64_t>(1, (n / (2 * pp) + kGmThreads - 1) / kGmThreads);
          auto* k3 = pp == 2 ? &k_gm_sweep_fast<3, 2> : &k_gm_sweep_fast<3, 1>;
          LAUNCH_PDL(c, k3, (unsigned)nsf[r], kGmThreads, 0, n, V, (const double*)d.gm[r].w.p,
                     (const GmDev*)d.gm[r].st.p, (const double*)nullptr, part, (const double*)vs(r), d.gm[r].V.p,
                     In.rk[r].buf.p);
        } else {
          nsf[r] = gm_blocks(n);
          LAUNCH_PDL(c, (k_gm_sweep<3, true>), (unsigned)nsf[r], kGmThreads, 0, n, V, d.gm[r].w.p,
                     (const GmDev*)d.gm[r].st.p, (const double*)nullptr, part, (const double*)vs(r), d.gm[r].V.p,
                     In.rk[r].buf.p, 1);
        }
        LAUNCH_PDL(c, k_gm_finish, 2 * kGmMax, kFinThreads, 0, (const double*)part, nsf[r],
                   (const GmDev*)d.gm[r].st.p, 0, dd(r));
      });
      allsum(2 * S, pd.p, dd);
      mine([&](int r) {
        LAUNCH_PDL(c, k_gm_gram, 1, 32, 0, (const GmDev*)d.gm[r].st.p, (const double*)dd(r), d.gm[r].G.p, h2(r),
                   hsum(r));
        const int64_t n = own(r);
        const int pp = n % 4 == 0 ? 2 : (n % 2 == 0 ? 1 : 0);
        double* part = d.gm[r].gpart.p;
        if (pp) {
          auto* k2 = pp == 2 ? &k_gm_sweep_fast<2, 2> : &k_gm_sweep_fast<2, 1>;
          LAUNCH_PDL(c, k2, (unsigned)nsf[r], kGmThreads, 0, n, (const double*)d.gm[r].V.p,
                     (const double*)d.gm[r].w.p, (const GmDev*)d.gm[r].st.p, (const double*)hsum(r), part,
                     (const double*)vs(r), d.gm[r].V.p, In.rk[r].buf.p);
        } else {
          LAUNCH_PDL(c, (k_gm_sweep<2, true>), (unsigned)nsf[r], kGmThreads, 0, n, (const double*)d.gm[r].V.p,
                     d.gm[r].w.p, (const GmDev*)d.gm[r].st.p, (const double*)hsum(r), part, (const double*)vs(r),
                     d.gm[r].V.p, In.rk[r].buf.p, 1);
        }
        LAUNCH_PDL(c, k_gm_finish, 1, kFinThreads, 0, (const double*)part, nsf[r], (const GmDev*)d.gm[r].st.p, 1,
                   nrm(r));
      });
      allsum(1, pn.p, nrm);
      mine([&](int r) {
        LAUNCH_PDL(c, k_gm_step, 1, 32, 0, 0, 0, d.gm[r].st.p, (const double*)dd(r), (const double*)h2(r),
                   (const double*)nrm(r), d.gm[r].H.p, d.gm[r].cs.p, d.gm[r].sn.p, d.gm[r].g.p, d.gm[r].hist.p,
                   vs(r));
      });
      // the lagged flag: this step's, read after the next step is enqueued
      CUDA_CHECK(cudaMemcpyAsync(d.gm_flag + (k & 1), &d.gm[rq].st.p->more, sizeof(int), cudaMemcpyDeviceToHost,
                                 c.stream));
      CUDA_CHECK(cudaEventRecord(ev[k & 1], c.stream));
      if (k >= 1) {
        CUDA_CHECK(cudaEventSynchronize(ev[(k - 1) & 1]));
        if (!d.gm_flag[(k - 1) & 1]) break;  // step k was past the end: a no-op
      }
      if (k + 1 >= m) break;  // the cycle's last column: no step past it
    }
    // ---- end of the cycle: y, x += Z y, r = b - A x, beta, the outer test
    mine([&](int r) {
      LAUNCH_PDL(c, k_gm_ysolve, 1, 32, 0, (const GmDev*)d.gm[r].st.p, (const double*)d.gm[r].H.p,
                 (const double*)d.gm[r].g.p, d.gm[r].y.p);
      if (own(r))
        LAUNCH_PDL(c, k_gm_xupdate, (unsigned)gm_blocks(own(r)), kGmThreads, 0, own(r), (const GmDev*)d.gm[r].st.p,
                   (const double*)d.gm[r].Z.p, (const double*)d.gm[r].y.p, d.gm[r].x.p);
    });
    stage_xs([&](int r) { return (const double*)d.gm[r].x.p; });
    mine([&](int r) {
      const Csr& A = d.rk[r].A0;
      if (!A.n) {
        CUDA_CHECK(cudaMemsetAsync(d.gm[r].sc.p, 0, sizeof(double), c.stream));
        return;
      }
      launch_rows(c, A, (const double*)d.XS.rk[r].buf.p,
                  LResid{d.rk[r].rhs.p, d.gm[r].w.p, d.part.p + d.part_off[r], 0.0}, false);
      const int np = (int)rows_grid(tview(A), false);
      LAUNCH_PDL(c, k_sum_part, 1, 1024, 0, (const double*)(d.part.p + d.part_off[r]), np, d.gm[r].sc.p);
    });
    release(c, d, d.XS);
    p2p_flush(c, d);
    allsum(1, ps.p, [&](int r) { return d.gm[r].sc.p; });
    mine([&](int r) { LAUNCH_PDL(c, k_gm_restart, 1, 32, 0, 0, 0, d.gm[r].st.p, (const double*)d.gm[r].sc.p); });
    to_host(c, &s1, d.gm[rq].st.p, 1);
    outer = !s1.converged && s1.beta != 0.0 && s1.its < s1.maxit;
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  (void)l0;
  to_host(c, &s1, d.gm[rq].st.p, 1);
  const long long kept = std::min<long long>(s1.its, cap - 1);
  std::vector<double> hv((size_t)kept + 1);
  to_host(c, hv.data(), d.gm[rq].hist.p, hv.size());
  for (double v : hv) hist.push_back(v);
  st.iterations = s1.its;
  st.converged = s1.converged;
  st.final_relative_residual = s1.rel;
  mine([&](int r) {
    const int64_t o = own(r), lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    if (o) CUDA_CHECK(cudaMemcpyAsync(d_x + lo, d.gm[r].x.p, sizeof(double) * o, cudaMemcpyDeviceToDevice, c.stream));
  });
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

void dist_gmres(Ctx& c, DHier& d, const airg_solve_config& cfg, const double* d_b, double* d_x,
                airg_solve_stats& st, std::vector<double>& hist) {
  const int L = (int)d.lv.size();
  const int P = d.P;
  const int m = (int)(cfg.gmres_restart > 0 ? cfg.gmres_restart : 30);
  if (m > 512) throw InvalidArgument("gmres: restart length above 512");
  static const bool host_gm = [] {
    const char* e = getenv("AIRG_DIST_GM_HOST");
    return e && e[0] == '1';
  }();
  if (m <= kGmMax && !host_gm && cfg.max_iterations > 0) {
    dist_gmres_dev(c, d, cfg, d_b, d_x, st, hist);
    return;
  }
  d.gm.clear();  // the host form allocates its own per-rank buffers
  DVec& In = L ? d.lv[0].B : d.CB;   // V-cycle input (owned part)
  DVec& Out = L ? d.lv[0].X : d.CX;  // V-cycle output (owned part)
  auto own = [&](int r) { return d.XS.rk[r].own; };
  if (d.gm_m != m || (int)d.gm.size() != P) {
    d.gm.clear();
    d.gm.resize(P);
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      const size_t o = (size_t)std::max<int64_t>(1, own(r));
      d.gm[r].V.alloc(c, o * (m + 1));
      d.gm[r].Z.alloc(c, o * m);
      d.gm[r].w.alloc(c, o);
      d.gm[r].x.alloc(c, o);
      d.gm[r].dots.alloc(c, (size_t)m + 2);
      d.gm[r].part.alloc(c, (size_t)(m + 2) * kGmDotBlocks);
    }
    d.gm_m = m;
  }
  const int64_t key = (cfg.up_f_smooths * 1000003 + cfg.coarse_iterations * 31) * 2 + (dist_fast(d, cfg) ? 1 : 0);
  if (!d.graph_vc || d.graph_vc_key != key) {
    d.graph_vc_kernels = capture_graph(c, &d.graph_vc, [&] {
      enqueue_vcycle(c, d, cfg);
      p2p_flush(c, d);
    });
    d.graph_vc_key = key;
  }
  // global sums of per-rank device scalars: rank order in emulation, one
  // NCCL allreduce per call with one rank per process
  auto allsum = [&](int cnt, const std::function<double*(int)>& dev) {
    std::vector<double> tot((size_t)cnt, 0.0), tmp((size_t)cnt);
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      double* p = dev(r);
      if (d.me >= 0 && P > 1) NCCL_CHECK(ncclAllReduce(p, p, (size_t)cnt, ncclDouble, ncclSum, d.comm, c.stream));
      to_host(c, tmp.data(), p, (size_t)cnt);
      for (int k = 0; k < cnt; ++k) tot[k] += tmp[k];
    }
    return tot;
  };
  auto local_dots = [&](int r, int jp1, const double* w) {
    const int64_t o = own(r);
    DHier::GmRank& G = d.gm[r];
    if (o)
      LAUNCH(c, k_gmd_dots, dim3(kGmDotBlocks, jp1), 256, 0, o, (const double*)G.V.p, w, G.part.p);
    else
      CUDA_CHECK(cudaMemsetAsync(G.part.p, 0, sizeof(double) * jp1 * kGmDotBlocks, c.stream));
    LAUNCH(c, k_gmd_fold, jp1, 32, 0, (const double*)G.part.p, kGmDotBlocks, G.dots.p);
  };
  // w = A x_in over the level-0 slabs (x_in: the owned part, staged in XS)
  auto matvec = [&](const std::function<const double*(int)>& xin, const std::function<double*(int)>& out,
                    bool resid) {
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r) || !own(r)) continue;
      CUDA_CHECK(cudaMemcpyAsync(d.XS.rk[r].buf.p, xin(r), sizeof(double) * own(r), cudaMemcpyDeviceToDevice,
                                 c.stream));
    }
    exchange(c, d, d.XS);
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      const Csr& A = d.rk[r].A0;
      if (!A.n) {
        CUDA_CHECK(cudaMemsetAsync(d.part.p + d.part_off[r], 0, sizeof(double), c.stream));
        continue;
      }
      if (resid)
        launch_rows(c, A, (const double*)d.XS.rk[r].buf.p, LResid{d.rk[r].rhs.p, out(r), d.part.p + d.part_off[r], 0.0});
      else
        launch_rows(c, A, (const double*)d.XS.rk[r].buf.p, LStore{out(r)});
    }
    release(c, d, d.XS);
    p2p_flush(c, d);
  };
  std::memset(&st, 0, sizeof st);
  const auto t0 = std::chrono::steady_clock::now();
  // b, x = 0, r = b
  for (int r = 0; r < P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t o = own(r), lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    if (o) {
      CUDA_CHECK(cudaMemcpyAsync(d.rk[r].rhs.p, d_b + lo, sizeof(double) * o, cudaMemcpyDeviceToDevice, c.stream));
      CUDA_CHECK(cudaMemcpyAsync(d.gm[r].w.p, d_b + lo, sizeof(double) * o, cudaMemcpyDeviceToDevice, c.stream));
    }
    CUDA_CHECK(cudaMemsetAsync(d.gm[r].x.p, 0, sizeof(double) * std::max<int64_t>(1, o), c.stream));
  }
  auto norm2 = [&](const std::function<const double*(int)>& v) {
    for (int r = 0; r < P; ++r) {
      if (!d.mine(r)) continue;
      const int64_t o = own(r);
      if (o)
        dot_async(c, v(r), v(r), o, d.gm[r].dots.p, d.gm[r].part.p);
      else
        CUDA_CHECK(cudaMemsetAsync(d.gm[r].dots.p, 0, sizeof(double), c.stream));
    }
    return allsum(1, [&](int r) { return d.gm[r].dots.p; })[0];
  };
  const double bnorm = std::sqrt(norm2([&](int r) { return (const double*)d.rk[r].rhs.p; }));
  int64_t its = 0;
  if (bnorm == 0.0) {
    st.converged = 1;
    hist.push_back(0.0);
  } else {
    double beta = bnorm;
    hist.push_back(1.0);
    st.final_relative_residual = 1.0;
    std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), hcol(m + 2), y(m + 1);
    while (its < cfg.max_iterations) {
      for (int r = 0; r < P; ++r)  // v_0 = r / beta, also the V-cycle input
        if (d.mine(r) && own(r))
          LAUNCH(c, k_gmd_scale, blocks_for(own(r), 256), 256, 0, own(r), (const double*)d.gm[r].w.p, 1.0 / beta,
                 d.gm[r].V.p, In.rk[r].buf.p);
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      for (; j < m && its < cfg.max_iterations; ++j) {
        CUDA_CHECK(cudaGraphLaunch(d.graph_vc, c.stream));
        c.launches += d.graph_vc_kernels;
        for (int r = 0; r < P; ++r)  // Z_j = M v_j
          if (d.mine(r) && own(r))
            CUDA_CHECK(cudaMemcpyAsync(d.gm[r].Z.p + (int64_t)j * own(r), Out.rk[r].buf.p, sizeof(double) * own(r),
                                       cudaMemcpyDeviceToDevice, c.stream));
        matvec([&](int r) { return (const double*)Out.rk[r].buf.p; }, [&](int r) { return d.gm[r].w.p; }, false);
        std::fill(hcol.begin(), hcol.end(), 0.0);
        for (int pass = 0; pass < 2; ++pass) {
          for (int r = 0; r < P; ++r)
            if (d.mine(r)) local_dots(r, j + 1, d.gm[r].w.p);
          const std::vector<double> hk = allsum(j + 1, [&](int r) { return d.gm[r].dots.p; });
          for (int r = 0; r < P; ++r) {
            if (!d.mine(r) || !own(r)) continue;
            to_device(c, d.gm[r].dots.p, hk.data(), hk.size());
            LAUNCH(c, k_gmd_update, blocks_for(own(r), 256), 256, 0, own(r), j + 1, (const double*)d.gm[r].V.p,
                   (const double*)d.gm[r].dots.p, d.gm[r].w.p);
          }
          for (int k = 0; k <= j; ++k) hcol[k] += hk[k];
        }
        const double hn = std::sqrt(norm2([&](int r) { return (const double*)d.gm[r].w.p; }));
        hcol[j + 1] = hn;
        for (int r = 0; r < P; ++r)
          if (d.mine(r) && own(r))
            LAUNCH(c, k_gmd_scale, blocks_for(own(r), 256), 256, 0, own(r), (const double*)d.gm[r].w.p,
                   hn > 0.0 ? 1.0 / hn : 0.0, d.gm[r].V.p + (int64_t)(j + 1) * own(r), In.rk[r].buf.p);
        for (int k = 0; k < j; ++k) {
          const double t = cs[k] * hcol[k] + sn[k] * hcol[k + 1];
          hcol[k + 1] = -sn[k] * hcol[k] + cs[k] * hcol[k + 1];
          hcol[k] = t;
        }
        const double den = std::hypot(hcol[j], hcol[j + 1]);
        cs[j] = den > 0.0 ? hcol[j] / den : 1.0;
        sn[j] = den > 0.0 ? hcol[j + 1] / den : 0.0;
        hcol[j] = den;
        hcol[j + 1] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        for (int k = 0; k <= j; ++k) H[k + (size_t)j * (m + 1)] = hcol[k];
        ++its;
        const double est = std::fabs(g[j + 1]) / bnorm;
        hist.push_back(est);
        if (est <= cfg.rtol || hn == 0.0) {
          ++j;
          break;
        }
      }
      for (int k = j - 1; k >= 0; --k) {
        double s = g[k];
        for (int q = k + 1; q < j; ++q) s -= H[k + (size_t)q * (m + 1)] * y[q];
        y[k] = s / H[k + (size_t)k * (m + 1)];
      }
      for (int r = 0; r < P; ++r) {
        if (!d.mine(r) || !own(r)) continue;
        to_device(c, d.gm[r].dots.p, y.data(), (size_t)j);
        LAUNCH(c, k_gmd_xupdate, blocks_for(own(r), 256), 256, 0, own(r), j, (const double*)d.gm[r].Z.p,
               (const double*)d.gm[r].dots.p, d.gm[r].x.p);
      }
      // r = b - A x (into w), beta = ||r||
      matvec([&](int r) { return (const double*)d.gm[r].x.p; }, [&](int r) { return d.gm[r].w.p; }, true);
      beta = std::sqrt(norm2([&](int r) { return (const double*)d.gm[r].w.p; }));
      const double rel = beta / bnorm;
      st.final_relative_residual = rel;
      if (rel <= cfg.rtol) {
        st.converged = 1;
        break;
      }
      if (beta == 0.0) break;
    }
  }
  for (int r = 0; r < P; ++r) {
    if (!d.mine(r) || !own(r)) continue;
    const int64_t lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    CUDA_CHECK(cudaMemcpyAsync(d_x + lo, d.gm[r].x.p, sizeof(double) * own(r), cudaMemcpyDeviceToDevice, c.stream));
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  st.iterations = its;
  st.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st.history_len = (int64_t)hist.size();
}

// Halo bytes this process receives per V-cycle (the exchanges of
// enqueue_vcycle, mine ranks only) and per level-0 SpMV (XS).
void dist_halo_bytes(const DHier& d, const airg_solve_config& cfg, int64_t& vcycle, int64_t& spmv) {
  auto halo = [&](const DVec& V) {
    int64_t s = 0;
    for (int r = 0; r < d.P; ++r)
      if (d.mine(r) && r < (int)V.rk.size()) s += V.rk[r].nhalo;
    return s;
  };
  const int L = (int)d.lv.size();
  const bool fast = dist_fast(d, cfg);
  int64_t e = 0;
  for (int l = 0; l < L; ++l) {
    const DLevel& D = d.lv[l];
    e += halo(D.B);                                        // restriction input
    e += halo(l + 1 < L ? d.lv[l + 1].X : d.CX);           // prolongation (fast: and A_F P) input
    if (fast)
      e += cfg.up_f_smooths > 0 ? halo(D.RF) : 0;          // W_k's input
    else
      e += cfg.up_f_smooths * (halo(D.X) + halo(D.RF));    // residual and update inputs
  }
  e += cfg.coarse_iterations * halo(d.CR) + std::max<int64_t>(0, cfg.coarse_iterations - 1) * halo(d.CX);
  vcycle = 8 * e;
  spmv = 8 * halo(d.XS);
}

void dist_solve(Ctx& c, DHier& d, const airg_solve_config& cfg, const double* d_b, double* d_x,
                airg_solve_stats& st, std::vector<double>& hist) {
  NvtxRange nvtx__("airg dist solve");
  if (cfg.down_smooths != 0) throw InvalidArgument("solve: down_smooths > 0 is not offered by the GPU V-cycle");
  dist_coarse_compose(c, d, cfg);
  if (cfg.rtol <= 0.0) throw InvalidArgument("richardson_solve: rtol must be positive");
  if (cfg.outer == 1) {
    dist_gmres(c, d, cfg, d_b, d_x, st, hist);
    return;
  }
  if (cfg.outer != 0) throw InvalidArgument("dist: outer must be 0 (Richardson) or 1 (GMRES)");
  std::memset(&st, 0, sizeof st);
  const int L = (int)d.lv.size();
  DVec& Rv = L ? d.lv[0].B : d.CB;
  const auto t0 = std::chrono::steady_clock::now();
  // scatter b (emulation: from the global vector; nccl: my slab)
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t own = d.XS.rk[r].own, lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    if (own) {
      CUDA_CHECK(cudaMemcpyAsync(d.rk[r].rhs.p, d_b + lo, sizeof(double) * own, cudaMemcpyDeviceToDevice, c.stream));
      CUDA_CHECK(cudaMemcpyAsync(Rv.rk[r].buf.p, d_b + lo, sizeof(double) * own, cudaMemcpyDeviceToDevice, c.stream));
    }
    CUDA_CHECK(cudaMemsetAsync(d.XS.rk[r].buf.p, 0, sizeof(double) * std::max<int64_t>(1, own), c.stream));
  }
  // ||b||: sum of local squared norms
  double bn2 = 0.0;
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t own = d.XS.rk[r].own;
    if (!own) continue;
    dot_async(c, d.rk[r].rhs.p, d.rk[r].rhs.p, own, d.scal.p + 1, d.part.p);
    bn2 += read1(c, d.scal.p + 1);
  }
  if (d.me >= 0 && d.P > 1) {
    to_device(c, d.scal.p + 2, &bn2, 1);
    bn2 = read_norm2(c, d, d.scal.p + 2);
  }
  const double bnorm = std::sqrt(bn2);
  if (bnorm == 0.0) {
    st.converged = 1;
    hist.push_back(0.0);
  } else {
    const int64_t key = (cfg.up_f_smooths * 1000003 + cfg.coarse_iterations * 31) * 2 + (dist_fast(d, cfg) ? 1 : 0);
    if (!d.graph || d.graph_key != key) {
      d.graph_kernels = capture_graph(c, &d.graph, [&] {
        enqueue_vcycle(c, d, cfg);
        enqueue_update_residual(c, d);
      });
      d.graph_key = key;
    }
    for (int64_t it = 0;; ++it) {
      const double rel = it == 0 ? 1.0 : std::sqrt(read_norm2(c, d, d.scal.p)) / bnorm;
      hist.push_back(rel);
      st.final_relative_residual = rel;
      if (rel <= cfg.rtol) {
        st.converged = 1;
        st.iterations = it;
        break;
      }
      if (it >= cfg.max_iterations) {
        st.iterations = it;
        break;
      }
      CUDA_CHECK(cudaGraphLaunch(d.graph, c.stream));
      c.launches += d.graph_kernels;
    }
  }
  for (int r = 0; r < d.P; ++r) {
    if (!d.mine(r)) continue;
    const int64_t own = d.XS.rk[r].own, lo = d.me < 0 ? d.XS.rk[r].lo : 0;
    if (own)
      CUDA_CHECK(cudaMemcpyAsync(d_x + lo, d.XS.rk[r].buf.p, sizeof(double) * own, cudaMemcpyDeviceToDevice,
                                 c.stream));
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  st.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st.history_len = (int64_t)hist.size();
}

}  // namespace airg
