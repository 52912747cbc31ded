// Scans and reductions used by the setup kernels and the solve.
#include "common.cuh"

namespace airg {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Exclusive scan of one 4096-element tile; writes tile-local exclusive
// prefixes and the tile total.
template <class Tin>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(const Tin* __restrict__ in,
                                                           int64_t* __restrict__ excl,
                                                           int64_t* __restrict__ tile_sum,
                                                           int64_t n) {
  __shared__ int64_t warp_sums[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? (int64_t)in[i] : 0;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = warp_incl_scan(s);
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t ws = warp_sums[lane];
    ws = warp_incl_scan(ws);
    warp_sums[lane] = ws;
  }
  __syncthreads();
  int64_t run = incl - s + (warp > 0 ? warp_sums[warp - 1] : 0);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < n) excl[i] = run;
    run += v[k];
  }
  if (threadIdx.x == kScanThreads - 1) tile_sum[blockIdx.x] = run;
}

template <class Tout>
__global__ void add_tile_offsets(const int64_t* __restrict__ excl,
                                 const int64_t* __restrict__ tile_off, Tout* __restrict__ out,
                                 int64_t n, const int64_t* __restrict__ total_src) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (Tout)(excl[i] + tile_off[i / kScanTile]);
  if (i == n) out[n] = (Tout)(*total_src);
}

// in-place exclusive scan of int64 values with the total appended at [n]
void scan64_inplace(Ctx& c, int64_t* d, int64_t n, int64_t* d_total) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  DBuf<int64_t> excl(c, (size_t)n), tsum(c, (size_t)tiles + 1);
  LAUNCH(c, scan_tiles<int64_t>, (unsigned)tiles, kScanThreads, 0, d, excl.p, tsum.p, n);
  if (tiles > 1) {
    scan64_inplace(c, tsum.p, tiles, d_total);
  } else {
    CUDA_CHECK(cudaMemcpyAsync(d_total, tsum.p, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    CUDA_CHECK(cudaMemsetAsync(tsum.p, 0, sizeof(int64_t), c.stream));
  }
  LAUNCH(c, add_tile_offsets<int64_t>, blocks_for(n + 1, 256), 256, 0, excl.p, tsum.p, d, n, d_total);
}

template <class Tin, class Tout>
int64_t scan_impl(Ctx& c, const Tin* d_counts, Tout* d_offsets, int64_t n) {
  DBuf<int64_t> total(c, 1);
  if (n == 0) {
    CUDA_CHECK(cudaMemsetAsync(d_offsets, 0, sizeof(Tout), c.stream));
    return 0;
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  DBuf<int64_t> excl(c, (size_t)n), tsum(c, (size_t)tiles + 1);
  LAUNCH(c, scan_tiles<Tin>, (unsigned)tiles, kScanThreads, 0, d_counts, excl.p, tsum.p, n);
  if (tiles > 1) {
    scan64_inplace(c, tsum.p, tiles, total.p);
  } else {
    CUDA_CHECK(cudaMemcpyAsync(total.p, tsum.p, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    CUDA_CHECK(cudaMemsetAsync(tsum.p, 0, sizeof(int64_t), c.stream));
  }
  LAUNCH(c, add_tile_offsets<Tout>, blocks_for(n + 1, 256), 256, 0, excl.p, tsum.p, d_offsets, n,
         total.p);
  return read1(c, total.p);
}

__global__ void dot_partials(const double* __restrict__ x, const double* __restrict__ y,
                             int64_t n, double* __restrict__ partials) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
  }
}

__global__ void reduce_partials(const double* __restrict__ partials, int np, double* out) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += partials[i];
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

void narrow_i64_to_i32(Ctx& c, const int64_t* in, int32_t* out, int64_t n);

int64_t exclusive_scan(Ctx& c, const int32_t* d_counts, int32_t* d_offsets, int64_t n) {
  // Scan in int64, then check the total fits the int32 offsets.
  DBuf<int64_t> off64(c, (size_t)n + 1);
  const int64_t total = scan_impl<int32_t, int64_t>(c, d_counts, off64.p, n);
  if (total > INT32_MAX) throw InvalidArgument("airg: nonzero count exceeds the int32 range");
  narrow_i64_to_i32(c, off64.p, d_offsets, n + 1);
  return total;
}

int64_t exclusive_scan64(Ctx& c, const int64_t* d_counts, int64_t* d_offsets, int64_t n) {
  return scan_impl<int64_t, int64_t>(c, d_counts, d_offsets, n);
}

namespace {
__global__ void narrow_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out,
                              int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)in[i];
}
}  // namespace

void narrow_i64_to_i32(Ctx& c, const int64_t* in, int32_t* out, int64_t n) {
  LAUNCH(c, narrow_kernel, blocks_for(n, 256), 256, 0, in, out, n);
}

void dot_async(Ctx& c, const double* x, const double* y, int64_t n, double* d_out,
               double* d_partials) {
  const int threads = 256;
  int blocks = (int)std::min<int64_t>(kReduceBlocks, (n + threads - 1) / threads);
  if (blocks < 1) blocks = 1;
  LAUNCH(c, dot_partials, blocks, threads, 0, x, y, n, d_partials);
  LAUNCH(c, reduce_partials, 1, 1024, 0, d_partials, blocks, d_out);
}

void csr_copy(Ctx& c, const Csr& a, Csr& out) {
  out.alloc(c, a.n, a.m, a.nnz);
  CUDA_CHECK(cudaMemcpyAsync(out.rp.p, a.rp.p, sizeof(int32_t) * (a.n + 1), cudaMemcpyDeviceToDevice, c.stream));
  if (a.nnz) {
    CUDA_CHECK(cudaMemcpyAsync(out.ci.p, a.ci.p, sizeof(int32_t) * a.nnz, cudaMemcpyDeviceToDevice, c.stream));
    CUDA_CHECK(cudaMemcpyAsync(out.v.p, a.v.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, c.stream));
  }
}

}  // namespace airg
