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

// Single-pass exclusive scan (decoupled look-back): one launch instead of
// tile scans + a scan of the tile sums + an offset pass (the setup runs
// about a thousand scans). Tiles of 4096 elements are taken in ticket order
// (a tile's predecessors are always already running). A tile publishes its
// aggregate, then its inclusive prefix, as ONE 64-bit descriptor word
// (status in bits 63..62: 0 empty, 1 aggregate, 2 prefix; the sum below), so
// no fence orders a flag against its value. Warp 0 looks back 32 tiles at a
// time. desc[0] is the ticket, desc[1 + t] tile t's descriptor (zeroed
// before the launch). out[n] and *total get the grand total. Integer sums:
// the result does not depend on the schedule.
constexpr unsigned long long kDescMask = (1ull << 62) - 1;
template <class Tin, class Tout>
__global__ void __launch_bounds__(kScanThreads) scan_lookback(const Tin* in, Tout* out, int64_t n,
                                                              unsigned long long* desc,
                                                              int64_t* __restrict__ total) {
  __shared__ int64_t warp_sums[kScanThreads / 32];
  __shared__ int64_t s_prefix;
  __shared__ unsigned s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd((unsigned*)desc, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    v[k] = i < n ? (int64_t)in[i] : 0;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t incl = warp_incl_scan(s);
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int64_t ws = warp_incl_scan(warp_sums[lane]);
    warp_sums[lane] = ws;
    const int64_t agg = __shfl_sync(0xffffffffu, ws, 31);  // the tile's total
    int64_t pre = 0;
    if (tile > 0) {
      if (lane == 0) atomicExch(desc + 1 + tile, (1ull << 62) | (unsigned long long)agg);
      int64_t look = tile - 1;
      while (true) {
        const int64_t t = look - lane;
        unsigned long long d = 2ull << 62;  // before tile 0: prefix 0
        if (t >= 0) {
          do {
            d = *(volatile unsigned long long*)(desc + 1 + t);
          } while ((d >> 62) == 0);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, (d >> 62) == 2);
        int64_t val = (int64_t)(d & kDescMask);
        if (pm && lane > __ffs(pm) - 1) val = 0;  // beyond the nearest prefix
#pragma unroll
        for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        pre += val;
        if (pm) break;
        look -= 32;
      }
    }
    if (lane == 0) {
      atomicExch(desc + 1 + tile, (2ull << 62) | (unsigned long long)(agg + pre));
      s_prefix = pre;
      if ((tile + 1) * kScanTile >= n) {  // the last tile
        out[n] = (Tout)(agg + pre);
        *total = agg + pre;
      }
    }
  }
  __syncthreads();
  int64_t run = incl - s + (warp > 0 ? warp_sums[warp - 1] : 0) + s_prefix;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = (Tout)run;
    run += v[k];
  }
}

template <class Tin, class Tout>
int64_t scan_impl(Ctx& c, const Tin* d_counts, Tout* d_offsets, int64_t n) {
  if (n == 0) {
    CUDA_CHECK(cudaMemsetAsync(d_offsets, 0, sizeof(Tout), c.stream));
    return 0;
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  DBuf<unsigned long long> desc(c, (size_t)tiles + 2);
  CUDA_CHECK(cudaMemsetAsync(desc.p, 0, sizeof(unsigned long long) * (size_t)(tiles + 2), c.stream));
  int64_t* total = (int64_t*)(desc.p + tiles + 1);
  LAUNCH(c, (scan_lookback<Tin, Tout>), (unsigned)tiles, kScanThreads, 0, d_counts, d_offsets, n, desc.p, total);
  return read1(c, total);
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

Ctx* ctx_workers(Ctx& c, int count) {
  if (c.n_workers >= count) return c.workers;
  Ctx* w = new Ctx[count];
  for (int k = 0; k < count; ++k) {
    if (k < c.n_workers) {
      w[k] = c.workers[k];
      continue;
    }
    w[k].device = c.device;
    w[k].num_sms = c.num_sms;
    CUDA_CHECK(cudaStreamCreateWithFlags(&w[k].own_stream, cudaStreamNonBlocking));
    w[k].stream = w[k].own_stream;
  }
  delete[] c.workers;
  c.workers = w;
  c.n_workers = count;
  return w;
}

bool setup_parallel(int part) {
  static const int mask = [] {
    const char* e = getenv("AIRG_SETUP_PARALLEL");
    return e ? atoi(e) : 1;
  }();
  return (mask & part) != 0;
}

void ctx_free_workers(Ctx& c) {
  for (int k = 0; k < c.n_workers; ++k) {
    Ctx& w = c.workers[k];
    cudaStreamSynchronize(w.stream);
    if (w.scratch) cudaFree(w.scratch);
    if (w.grid_bar) cudaFree(w.grid_bar);
    if (w.pinned) cudaFreeHost(w.pinned);
    if (w.own_stream) cudaStreamDestroy(w.own_stream);
  }
  delete[] c.workers;
  c.workers = nullptr;
  c.n_workers = 0;
}

int64_t exclusive_scan(Ctx& c, const int32_t* d_counts, int32_t* d_offsets, int64_t n) {
  // Summed in int64 (the offsets are narrowed as they are written): a total
  // beyond the int32 offsets is refused before anything reads them.
  const int64_t total = scan_impl<int32_t, int32_t>(c, d_counts, d_offsets, n);
  if (total > INT32_MAX) throw InvalidArgument("airg: nonzero count exceeds the int32 range");
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
