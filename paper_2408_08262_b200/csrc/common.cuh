// Shared infrastructure of the B200 AIRG engine: status/exception plumbing,
// the context (device, stream, launch counter), stream-ordered device
// buffers, the device CSR type and scan / reduction helpers.
//
// Arithmetic policy: the whole library is compiled with --fmad=false, so
// every a*b+c the reference writes as a separate multiply and add is
// rounded twice exactly as on the host (the reference is built without FMA,
// SURVEY §0.3). Kernels that must be bit-identical to the reference keep its
// per-row sequential accumulation order (thread-per-row). Explicit fma()
// calls (double-double arithmetic) are unaffected by --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "airg_c.h"

namespace airg {

// NVTX range for the phases a profiler should see (header-only NVTX3: a
// no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------------------
// errors: C++ exceptions inside the library, mapped to status codes at the
// C-ABI boundary (capi.cu) the way cli.cpp:477-486 maps the reference's.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // a non-sticky error must not resurface at the next launch check
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    throw CudaError(buf);
  }
}
#define CUDA_CHECK(x) ::airg::cuda_check((x), #x, __FILE__, __LINE__)

// reference counter RNG (rng.hpp:13-24), host side
inline uint64_t splitmix64_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t mix_host(uint64_t seed, uint64_t key) {
  return splitmix64_host(seed ^ splitmix64_host(key));
}

// ---------------------------------------------------------------------------
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  uint64_t launches = 0;
  int num_sms = 148;
  // pinned host staging for small readbacks (allocated on first use)
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // reusable device scratch (stream-ordered; grown on demand)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // software grid-barrier words of persistent kernels (self-resetting)
  unsigned* grid_bar = nullptr;
  // worker contexts (ctx_workers): own streams and staging on the same
  // device, for independent chains enqueued side by side by host threads
  Ctx* workers = nullptr;
  int n_workers = 0;
};

// `count` worker contexts of c (created on first use, kept until the context
// is destroyed). A worker's stream is not ordered against c.stream: the
// caller synchronises c.stream before handing work out and every worker's
// stream before taking results back.
Ctx* ctx_workers(Ctx& c, int count);
// Independent setup chains enqueued side by side by host threads on worker
// streams: 1 = a level's retry fits, 2 = the levels' fused operators, 4 = P
// and A P beside the inverse fit. AIRG_SETUP_PARALLEL=<mask>; 0: everything
// on the context's stream, one chain after the other. Default 1. Measured on
// C4 (B200): 0 -> 87 ms setup, 1 -> 78 ms, 7 -> 66 ms -- but after a setup
// with part 2 or 4 every device-resident solve loop (the conditional WHILE
// graphs of GMRES and Richardson) runs ~15 us per iteration slower (C4 solve
// 67.8 -> 70.1 ms) although each kernel, launched one by one, takes the same
// time, wherever the operators and the Krylov basis are placed (one arena,
// fresh cudaMalloc) and whether or not the worker streams still exist: the
// solve is the metric, so parts 2 and 4 are opt-in for setup-bound uses.
bool setup_parallel(int part);
void ctx_free_workers(Ctx& c);

// Device scratch of at least `bytes` (contents undefined), reused across
// calls on the context's stream.
inline void* ctx_scratch(Ctx& c, size_t bytes);

// Launch helper: counts every kernel this library enqueues (bench.py reports
// the delta as gpu_launches) and checks the launch.
#define LAUNCH(ctx, kernel, grid, block, smem, ...)                                   \
  do {                                                                                \
    (ctx).launches++;                                                                 \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);                   \
    CUDA_CHECK(cudaGetLastError());                                                   \
  } while (0)

// Programmatic dependent launch (sm_90+): a kernel launched with
// LAUNCH_PDL may start while its predecessor drains; it must call
// pdl_wait() before touching anything the predecessor writes, and calls
// pdl_trigger() to let its own successor launch early. Both are no-ops for
// ordinary launches.
// L2 eviction priority of a load stream (createpolicy + ld ... L2::cache_hint):
// 1 = evict_first (the Krylov basis, streamed by the GMRES sweeps), else
// evict_last. (Per-level priorities on the V-cycle operators -- evict_first
// for the fine levels, evict_last for the coarse tail -- measured neutral to
// 1.5 % slower on C4.)
__device__ __forceinline__ unsigned long long l2_policy(int hint) {
  unsigned long long p;
  if (hint == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
  double d;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(a), "l"(pol));
  return d;
}
__device__ __forceinline__ double2 ld2_hint(const double* a, unsigned long long pol) {
  double2 d;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(d.x), "=d"(d.y) : "l"(a), "l"(pol));
  return d;
}
__device__ __forceinline__ int ld_hint(const int* a, unsigned long long pol) {
  int d;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(d) : "l"(a), "l"(pol));
  return d;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
inline void launch_pdl(Ctx& c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  static const bool enabled = [] {
    const char* e = getenv("AIRG_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = enabled ? 1 : 0;
  c.launches++;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}
#define LAUNCH_PDL(ctx, kernel, grid, block, smem, ...) \
  ::airg::launch_pdl((ctx), kernel, dim3(grid), dim3(block), (smem), __VA_ARGS__)

// one atomic per block: warp shuffles, then the block's warps through shared
// memory (counters shared by all rows would otherwise serialise at L2)
__device__ __forceinline__ void block_add(unsigned long long* dst, unsigned long long v) {
  __shared__ unsigned long long part[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    if (t) atomicAdd(dst, t);
  }
}
__device__ __forceinline__ void block_max(unsigned long long* dst, unsigned long long v) {
  __shared__ unsigned long long part[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = max(t, part[w]);
    if (t) atomicMax(dst, t);
  }
}


// Sense-free grid barrier over co-resident CTAs: bar[0] arrivals, bar[1]
// generation. The last CTA to arrive resets the count and bumps the
// generation; the others spin on it (bounded: a lost CTA traps instead of
// hanging the device).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned spins = 0;
      while (*gen == g) {
        if (++spins > (1u << 30)) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}


inline unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------
// Stream-ordered device buffer (cudaMallocAsync from the default pool, whose
// release threshold is raised at context creation so frees are cached).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool borrowed = false;  // a view into memory owned elsewhere (never freed here)

  DBuf() = default;
  DBuf(Ctx& c, size_t count) { alloc(c, count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), borrowed(o.borrowed) {
    o.p = nullptr;
    o.n = 0;
    o.borrowed = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; borrowed = o.borrowed;
      o.p = nullptr; o.n = 0; o.borrowed = false;
    }
    return *this;
  }
  void view(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
    borrowed = true;
  }
  ~DBuf() { release(); }

  void alloc(Ctx& c, size_t count) {
    release();
    s = c.stream;
    n = count;
    if (count) {
      cudaError_t e = cudaMallocAsync((void**)&p, count * sizeof(T), s);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        p = nullptr;
        n = 0;
        char buf[128];
        snprintf(buf, sizeof buf, "device allocation of %zu bytes failed", count * sizeof(T));
        throw CudaError(buf);
      }
    }
  }
  void release() {
    if (p && !borrowed) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    borrowed = false;
  }
  void zero(Ctx& c) {
    if (n) CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), c.stream));
  }
  T* get() const { return p; }
};

inline void* ctx_scratch(Ctx& c, size_t bytes) {
  if (bytes > c.scratch_bytes) {
    if (c.scratch) CUDA_CHECK(cudaFreeAsync(c.scratch, c.stream));
    const size_t want = std::max(bytes, 2 * c.scratch_bytes);
    CUDA_CHECK(cudaMallocAsync(&c.scratch, want, c.stream));
    c.scratch_bytes = want;
  }
  return c.scratch;
}

// Read a few values back (synchronises the context stream). Small reads go
// through a pinned staging buffer: a pageable D2H copy costs a staged,
// synchronous transfer.
constexpr size_t kPinnedBytes = 1 << 16;
template <class T>
inline void to_host(Ctx& c, T* h, const T* d, size_t count) {
  if (!count) return;
  const size_t bytes = count * sizeof(T);
  if (bytes <= kPinnedBytes) {
    if (!c.pinned) {
      CUDA_CHECK(cudaMallocHost(&c.pinned, kPinnedBytes));
      c.pinned_bytes = kPinnedBytes;
    }
    CUDA_CHECK(cudaMemcpyAsync(c.pinned, d, bytes, cudaMemcpyDeviceToHost, c.stream));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    std::memcpy(h, c.pinned, bytes);
    return;
  }
  CUDA_CHECK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c.stream));
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
}
template <class T>
inline T read1(Ctx& c, const T* d) {
  T v;
  to_host(c, &v, d, 1);
  return v;
}
template <class T>
inline void to_device(Ctx& c, T* d, const T* h, size_t count) {
  if (!count) return;
  CUDA_CHECK(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, c.stream));
}

// ---------------------------------------------------------------------------
// Device CSR: int32 offsets / columns, fp64 values (12 B per nonzero).
struct Csr {
  int32_t n = 0, m = 0;
  int64_t nnz = 0;
  int32_t max_row = -1;  // longest row, when measured (row_max; sizes the fast row kernels)
  DBuf<int32_t> rp, ci;
  DBuf<double> v;

  Csr() = default;
  Csr(Csr&&) = default;
  Csr& operator=(Csr&&) = default;
  void alloc(Ctx& c, int64_t rows, int64_t cols, int64_t nz) {
    if (rows > INT32_MAX || cols > INT32_MAX || nz > INT32_MAX)
      throw InvalidArgument("airg: matrix exceeds the int32 device index range");
    n = (int32_t)rows;
    m = (int32_t)cols;
    nnz = nz;
    rp.alloc(c, (size_t)rows + 1);
    ci.alloc(c, (size_t)nz);
    v.alloc(c, (size_t)nz);
  }
};

// ---------------------------------------------------------------------------
// helpers implemented in util.cu
// exclusive scan of int32 counts into int32 offsets[n+1]; returns the total
// (checked against the int32 range).
int64_t exclusive_scan(Ctx& c, const int32_t* d_counts, int32_t* d_offsets, int64_t n);
// same for int64 counts/offsets
int64_t exclusive_scan64(Ctx& c, const int64_t* d_counts, int64_t* d_offsets, int64_t n);
// parallel dot product / squared norm (not order-preserving), result on device
void dot_async(Ctx& c, const double* x, const double* y, int64_t n, double* d_out,
               double* d_partials);
constexpr int kReduceBlocks = 1184;  // 8 x 148 SMs

// Copy a CSR (device -> device)
void csr_copy(Ctx& c, const Csr& a, Csr& out);

}  // namespace airg
