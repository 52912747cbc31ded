// airgraph_gpu.hpp -- C++ drop-in adapter over include/airg_c.h.
//
// Lets code written against the reference library (namespace airgraph,
// /root/reference/proj/include/airgraph/*.hpp) hand its own value types to
// the B200 engine. Matrix types are duck-typed templates: anything with
// nrows(), ncols(), row_offsets(), col_indices(), values() and a
// (nrows, ncols, offsets, cols, values) constructor -- exactly
// airgraph::SparseMatrix (sparse.hpp:33-94). Errors come back as the
// reference's exception types: std::invalid_argument for AIRG_EINVAL,
// std::runtime_error for everything else (cli.cpp:477-486 mapping).
//
// Header-only; link libairg_b200.so.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "airg_c.h"

namespace airgraph_gpu {

inline void check(int rc) {
  if (rc == AIRG_OK) return;
  char buf[4096];
  airg_last_error(buf, sizeof buf);
  if (rc == AIRG_EINVAL) throw std::invalid_argument(buf);
  throw std::runtime_error(buf);
}

class Context {
 public:
  explicit Context(int device = 0) { check(airg_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) airg_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  airg_ctx* get() const { return h_; }

 private:
  airg_ctx* h_ = nullptr;
};

class Matrix {
 public:
  Matrix() = default;
  explicit Matrix(airg_csr* h, bool owned = true) : h_(h), owned_(owned) {}
  Matrix(Matrix&& o) noexcept : h_(o.h_), owned_(o.owned_) { o.h_ = nullptr; }
  Matrix& operator=(Matrix&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(owned_, o.owned_);
    return *this;
  }
  ~Matrix() {
    if (h_ && owned_) airg_csr_destroy(h_);
  }
  const airg_csr* get() const { return h_; }
  int64_t nrows() const { return dims()[0]; }
  int64_t ncols() const { return dims()[1]; }
  int64_t nnz() const { return dims()[2]; }

 private:
  std::vector<int64_t> dims() const {
    int64_t n, m, z;
    check(airg_csr_info(h_, &n, &m, &z));
    return {n, m, z};
  }
  airg_csr* h_ = nullptr;
  bool owned_ = true;
};

// Reference SparseMatrix -> device (validating, sparse.cpp:18-46 checks).
template <class SM>
Matrix upload(Context& ctx, const SM& a) {
  airg_csr* h = nullptr;
  check(airg_csr_upload(ctx.get(), a.nrows(), a.ncols(), a.row_offsets().data(),
                        a.col_indices().data(), a.values().data(), &h));
  return Matrix(h);
}

// device -> reference SparseMatrix (value semantics, like every reference result)
template <class SM>
SM download(Context& ctx, const Matrix& m) {
  using index_t = typename std::decay_t<decltype(std::declval<SM>().row_offsets())>::value_type;
  const int64_t n = m.nrows(), c = m.ncols(), z = m.nnz();
  std::vector<int64_t> rp(n + 1), ci(z);
  std::vector<double> v(z);
  check(airg_csr_download(ctx.get(), m.get(), rp.data(), ci.data(), v.data()));
  return SM(n, c, std::vector<index_t>(rp.begin(), rp.end()),
            std::vector<index_t>(ci.begin(), ci.end()), std::move(v));
}

// airgraph::spmv (sparse.hpp:97-98) with host vectors.
template <class SM>
std::vector<double> spmv(Context& ctx, const SM& a, std::span<const double> x) {
  if ((int64_t)x.size() != (int64_t)a.ncols()) throw std::invalid_argument("spmv: dimension mismatch");
  Matrix d = upload(ctx, a);
  std::vector<double> y(a.nrows());
  check(airg_spmv_host(ctx.get(), d.get(), x.data(), y.data()));
  return y;
}

// airgraph::spgemm (sparse.hpp:101)
template <class SM>
SM spgemm(Context& ctx, const SM& a, const SM& b) {
  Matrix da = upload(ctx, a), db = upload(ctx, b);
  airg_csr* out = nullptr;
  check(airg_spgemm(ctx.get(), da.get(), db.get(), &out));
  return download<SM>(ctx, Matrix(out));
}

// airgraph::drop_entries (sparse.hpp:109-110)
template <class SM>
SM drop_entries(Context& ctx, const SM& a, double tol, bool keep_diagonal = true) {
  Matrix da = upload(ctx, a);
  airg_csr* out = nullptr;
  check(airg_drop(ctx.get(), da.get(), tol, keep_diagonal ? 1 : 0, &out));
  return download<SM>(ctx, Matrix(out));
}

// strength -> pmisr -> extract_blocks -> ddc (air.cpp:466-494), labels as
// airgraph::CfLabel values (F = 0, C = 1).
template <class SM>
std::vector<uint8_t> cf_split(Context& ctx, const SM& a, double alpha, int64_t max_loops,
                              uint64_t seed, bool ddc_enabled = true, double ddc_fraction = 0.1,
                              int64_t ddc_bins = 1000, airg_cf_report* report = nullptr) {
  Matrix d = upload(ctx, a);
  std::vector<uint8_t> labels(a.nrows());
  airg_cf_report rep;
  check(airg_cf_split_host(ctx.get(), d.get(), alpha, max_loops, seed, 0, ddc_enabled ? 1 : 0,
                           ddc_fraction, ddc_bins, labels.data(), &rep));
  if (report) *report = rep;
  return labels;
}

// device scratch through the C-ABI (no CUDA runtime needed on this side)
class DeviceBuffer {
 public:
  DeviceBuffer(Context& ctx, size_t bytes) : ctx_(&ctx) { check(airg_device_alloc(ctx.get(), bytes, &p_)); }
  ~DeviceBuffer() {
    if (p_) airg_device_free(ctx_->get(), p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ctx_(o.ctx_), p_(o.p_) { o.p_ = nullptr; }
  template <class T>
  T* as() const { return static_cast<T*>(p_); }
  void upload(const void* h, size_t bytes) { check(airg_memcpy(ctx_->get(), p_, h, bytes, 1)); }
  void download(void* h, size_t bytes) const { check(airg_memcpy(ctx_->get(), h, p_, bytes, 0)); }

 private:
  Context* ctx_;
  void* p_ = nullptr;
};

// dominance_report (coarsening.hpp:106): theta per A_ff row, histogram, max
struct DominanceReport {
  std::vector<double> theta;
  double max_theta = 0.0;
  std::vector<int64_t> histogram;
};
template <class SM>
DominanceReport dominance_report(Context& ctx, const SM& a_ff, int64_t bins = 1000) {
  Matrix d = upload(ctx, a_ff);
  DominanceReport r;
  r.theta.resize(a_ff.nrows());
  r.histogram.assign(bins > 0 ? bins : 0, 0);
  DeviceBuffer dt(ctx, sizeof(double) * r.theta.size());
  check(airg_dominance_report(ctx.get(), d.get(), bins, dt.as<double>(), r.histogram.data(), &r.max_theta));
  dt.download(r.theta.data(), sizeof(double) * r.theta.size());
  return r;
}

// apply_polynomial (gmres_poly.hpp:40-43): q(A) b, coefficients[0..eff]
template <class SM>
std::vector<double> apply_polynomial(Context& ctx, const SM& a, std::span<const double> coeffs, int64_t eff,
                                     std::span<const double> b) {
  if ((int64_t)b.size() != a.ncols()) throw std::invalid_argument("apply_polynomial: dimension mismatch");
  Matrix d = upload(ctx, a);
  const size_t n = a.nrows();
  DeviceBuffer db(ctx, sizeof(double) * b.size()), dy(ctx, sizeof(double) * n);
  db.upload(b.data(), sizeof(double) * b.size());
  check(airg_apply_polynomial(ctx.get(), d.get(), coeffs.data(), (int64_t)coeffs.size(), eff, db.as<double>(),
                              dy.as<double>()));
  std::vector<double> y(n);
  dy.download(y.data(), sizeof(double) * n);
  return y;
}

// build_restriction (air.hpp:96-98); labels as airgraph::CfLabel values (F = 0, C = 1)
template <class SM>
SM build_restriction(Context& ctx, const SM& a_cf, const SM& aff_inv, double drop_restrict,
                     const std::vector<uint8_t>& labels) {
  Matrix dcf = upload(ctx, a_cf), dinv = upload(ctx, aff_inv);
  DeviceBuffer dl(ctx, labels.size());
  dl.upload(labels.data(), labels.size());
  airg_csr* out = nullptr;
  check(airg_build_restriction(ctx.get(), dcf.get(), dinv.get(), drop_restrict, dl.as<uint8_t>(),
                               (int64_t)labels.size(), &out));
  return download<SM>(ctx, Matrix(out));
}

// build_prolongation (air.hpp:104-105) with g given as the strength pattern S
template <class SM>
SM build_prolongation(Context& ctx, const SM& a, const SM& s_pattern, const std::vector<uint8_t>& labels) {
  Matrix da = upload(ctx, a), ds = upload(ctx, s_pattern);
  DeviceBuffer dl(ctx, labels.size());
  dl.upload(labels.data(), labels.size());
  airg_csr* out = nullptr;
  check(airg_build_prolongation(ctx.get(), da.get(), ds.get(), dl.as<uint8_t>(), &out));
  return download<SM>(ctx, Matrix(out));
}

// coarse_matrix (air.hpp:113-114): drop_entries(R (A P), drop_coarse)
template <class SM>
SM coarse_matrix(Context& ctx, const SM& r, const SM& a, const SM& p, double drop_coarse) {
  Matrix dr = upload(ctx, r), da = upload(ctx, a), dp = upload(ctx, p);
  airg_csr* out = nullptr;
  check(airg_coarse_matrix(ctx.get(), dr.get(), da.get(), dp.get(), drop_coarse, &out));
  return download<SM>(ctx, Matrix(out));
}

// airgraph::setup (air.hpp:126) -> a device-resident hierarchy
class Hierarchy {
 public:
  template <class SM>
  Hierarchy(Context& ctx, const SM& a, const airg_setup_config& cfg,
            const airg_injection* inj = nullptr)
      : ctx_(&ctx) {
    Matrix d = upload(ctx, a);
    check(airg_setup(ctx.get(), d.get(), &cfg, inj, &h_));
    top_n_ = a.nrows();
  }
  ~Hierarchy() {
    if (h_) airg_hier_destroy(h_);
  }
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;
  airg_hier_info info() const {
    airg_hier_info i;
    check(airg_hier_info_get(h_, &i));
    return i;
  }
  std::vector<uint8_t> labels(int64_t level) const {
    airg_level_info li;
    check(airg_hier_level_info(h_, level, &li));
    std::vector<uint8_t> out(li.n);
    check(airg_hier_labels(ctx_->get(), h_, level, out.data()));
    return out;
  }
  // airgraph::richardson_solve (solve.hpp:60-61) / outer GMRES (cfg.outer = 1)
  airg_solve_stats solve(std::span<const double> b, std::vector<double>* x_out,
                         const airg_solve_config& cfg,
                         std::vector<double>* history = nullptr) const {
    if ((int64_t)b.size() != top_n_) throw std::invalid_argument("richardson_solve: rhs length mismatch");
    std::vector<double> x(b.size());
    std::vector<double> hist(history ? 4096 : 0);
    airg_solve_stats st;
    check(airg_solve_host(ctx_->get(), h_, &cfg, b.data(), x.data(), &st,
                          history ? hist.data() : nullptr, (int64_t)hist.size()));
    if (history) {
      hist.resize(std::min<int64_t>(st.history_len, (int64_t)hist.size()));
      *history = std::move(hist);
    }
    if (x_out) *x_out = std::move(x);
    return st;
  }

 private:
  Context* ctx_;
  airg_hier* h_ = nullptr;
  int64_t top_n_ = 0;
};

}  // namespace airgraph_gpu
