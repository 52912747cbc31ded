// Row-partitioned setup work (see rowsplit.cuh).
#include <algorithm>

#include "rowsplit.cuh"

namespace airg {

#define RS_NCCL(x)                                                             \
  do {                                                                         \
    ncclResult_t r__ = (x);                                                    \
    if (r__ != ncclSuccess)                                                    \
      throw CudaError(std::string("NCCL error: ") + ncclGetErrorString(r__)); \
  } while (0)

namespace {

__global__ void k_slice_rows(int n_local, int64_t row0, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, const double* __restrict__ v,
                             int32_t* __restrict__ orp, int32_t* __restrict__ oci, double* __restrict__ ov) {
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

// out.rp[row0 + i] = rp[i] + off for the rows of one slab
__global__ void k_place_rp(int n_local, int64_t row0, int64_t off, const int32_t* __restrict__ rp,
                           int32_t* __restrict__ orp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_local) orp[row0 + i] = (int32_t)(rp[i] + off);
}

template <class T>
ncclDataType_t nccl_type();
template <>
ncclDataType_t nccl_type<double>() { return ncclDouble; }
template <>
ncclDataType_t nccl_type<int32_t>() { return ncclInt32; }
template <>
ncclDataType_t nccl_type<uint8_t>() { return ncclUint8; }

template <class T>
void gather_impl(Ctx& c, const RowSplit& rs, T* y, const std::vector<int64_t>& s) {
  if (rs.me < 0 || rs.P == 1) return;  // emulation: every slab was written in place
  RS_NCCL(ncclGroupStart());
  for (int r = 0; r < rs.P; ++r) {
    const int64_t n = s[r + 1] - s[r];
    if (n > 0) RS_NCCL(ncclBroadcast(y + s[r], y + s[r], (size_t)n, nccl_type<T>(), r, rs.comm, c.stream));
  }
  RS_NCCL(ncclGroupEnd());
}

}  // namespace

std::vector<int64_t> RowSplit::slabs(int64_t n) const {
  std::vector<int64_t> s((size_t)P + 1, 0);
  const int64_t base = n / P, extra = n % P;
  for (int r = 0; r < P; ++r) s[r + 1] = s[r] + base + (r < extra ? 1 : 0);
  return s;
}

void RowSplit::gather_vec(Ctx& c, double* y, const std::vector<int64_t>& s) const { gather_impl(c, *this, y, s); }
void RowSplit::gather_vec(Ctx& c, int32_t* y, const std::vector<int64_t>& s) const { gather_impl(c, *this, y, s); }
void RowSplit::gather_vec(Ctx& c, uint8_t* y, const std::vector<int64_t>& s) const { gather_impl(c, *this, y, s); }

void csr_slice(Ctx& c, const Csr& a, int64_t lo, int64_t hi, Csr& out) {
  const int64_t n = hi - lo;
  int32_t b[2] = {0, 0};
  if (n > 0) {
    to_host(c, &b[0], a.rp.p + lo, 1);
    to_host(c, &b[1], a.rp.p + hi, 1);
  }
  out.alloc(c, n, a.m, b[1] - b[0]);
  if (n > 0)
    LAUNCH(c, k_slice_rows, blocks_for(n + 1, 256), 256, 0, (int)n, lo, a.rp.p, a.ci.p, a.v.p, out.rp.p,
           out.ci.p, out.v.p);
  else
    out.rp.zero(c);
}

void RowSlices::build(Ctx& c, const RowSplit& rs, const Csr& a) {
  s = rs.slabs(a.n);
  part.clear();
  part.resize(rs.P);
  for (int r = 0; r < rs.P; ++r)
    if (rs.mine(r)) csr_slice(c, a, s[r], s[r + 1], part[r]);
}

void split_spmv(Ctx& c, const RowSplit& rs, const RowSlices& a, const double* x, double* y) {
  for (int r = 0; r < rs.P; ++r)
    if (rs.mine(r) && a.part[r].n) spmv(c, a.part[r], x, y + a.s[r]);
  rs.gather_vec(c, y, a.s);
}

void gather_csr(Ctx& c, const RowSplit& rs, const std::vector<int64_t>& s, std::vector<Csr>& slab,
                int64_t ncols, Csr& out) {
  const int P = rs.P;
  const int64_t n = s[P];
  // nnz of every slab on every rank
  std::vector<int64_t> nnz(P, 0);
  if (rs.me < 0) {
    for (int r = 0; r < P; ++r) nnz[r] = slab[r].nnz;
  } else {
    DBuf<int64_t> cnt(c, (size_t)P);
    cnt.zero(c);
    const int64_t mine = slab[rs.me].nnz;
    to_device(c, cnt.p + rs.me, &mine, 1);
    if (P > 1) {
      RS_NCCL(ncclGroupStart());
      for (int r = 0; r < P; ++r) RS_NCCL(ncclBroadcast(cnt.p + r, cnt.p + r, 1, ncclInt64, r, rs.comm, c.stream));
      RS_NCCL(ncclGroupEnd());
    }
    to_host(c, nnz.data(), cnt.p, (size_t)P);
  }
  std::vector<int64_t> off(P + 1, 0);
  for (int r = 0; r < P; ++r) off[r + 1] = off[r] + nnz[r];
  out.alloc(c, n, ncols, off[P]);
  const int32_t total = (int32_t)off[P];
  to_device(c, out.rp.p + n, &total, 1);
  for (int r = 0; r < P; ++r) {
    if (!rs.mine(r)) continue;
    const int64_t nr = s[r + 1] - s[r];
    if (nr > 0)
      LAUNCH(c, k_place_rp, blocks_for(nr, 256), 256, 0, (int)nr, s[r], off[r], slab[r].rp.p, out.rp.p);
    if (nnz[r]) {
      CUDA_CHECK(cudaMemcpyAsync(out.ci.p + off[r], slab[r].ci.p, sizeof(int32_t) * nnz[r],
                                 cudaMemcpyDeviceToDevice, c.stream));
      CUDA_CHECK(cudaMemcpyAsync(out.v.p + off[r], slab[r].v.p, sizeof(double) * nnz[r],
                                 cudaMemcpyDeviceToDevice, c.stream));
    }
  }
  if (rs.me >= 0 && P > 1) {
    RS_NCCL(ncclGroupStart());
    for (int r = 0; r < P; ++r) {
      const int64_t nr = s[r + 1] - s[r];
      if (nr > 0) RS_NCCL(ncclBroadcast(out.rp.p + s[r], out.rp.p + s[r], (size_t)nr, ncclInt32, r, rs.comm, c.stream));
      if (nnz[r]) {
        RS_NCCL(ncclBroadcast(out.ci.p + off[r], out.ci.p + off[r], (size_t)nnz[r], ncclInt32, r, rs.comm, c.stream));
        RS_NCCL(ncclBroadcast(out.v.p + off[r], out.v.p + off[r], (size_t)nnz[r], ncclDouble, r, rs.comm, c.stream));
      }
    }
    RS_NCCL(ncclGroupEnd());
  }
}

void split_spgemm(Ctx& c, const RowSplit& rs, const Csr& a, const Csr& b, Csr& out, double drop_tol,
                  bool keep_diag) {
  const std::vector<int64_t> s = rs.slabs(a.n);
  std::vector<Csr> slab(rs.P);
  for (int r = 0; r < rs.P; ++r) {
    if (!rs.mine(r)) continue;
    Csr ar;
    csr_slice(c, a, s[r], s[r + 1], ar);
    spgemm(c, ar, b, slab[r], drop_tol, keep_diag, nullptr, (int)s[r], a.n);
  }
  gather_csr(c, rs, s, slab, b.m, out);
}

}  // namespace airg
