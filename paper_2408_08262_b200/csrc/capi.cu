// extern "C" boundary (include/airg_c.h): status codes + thread-local error
// text, mirroring how the reference surfaces std::invalid_argument /
// std::runtime_error (cli.cpp:477-486).
#include <cstring>
#include <memory>

#include "dist.cuh"
#include "mmio.cuh"
#include "rowsplit.cuh"

using namespace airg;

struct airg_ctx {
  Ctx c;
};
struct airg_csr {
  Ctx* c = nullptr;
  Csr m;
};
struct airg_hier {
  Ctx* c = nullptr;
  Hier h;
  std::vector<std::unique_ptr<airg_csr>> views;  // borrowed handles
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return AIRG_OK;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return AIRG_EINVAL;
  } catch (const RuntimeError& e) {
    g_err = e.what();
    return AIRG_ERUNTIME;
  } catch (const CudaError& e) {
    g_err = e.what();
    return AIRG_ECUDA;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return AIRG_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return AIRG_ELOGIC;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw InvalidArgument(std::string("airg: null ") + what);
}
void bind(Ctx& c) { CUDA_CHECK(cudaSetDevice(c.device)); }

}  // namespace

extern "C" {

int airg_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)g_err.size();
}

const char* airg_version(void) { return "airg-b200 0.1 (sm_100a)"; }

void airg_setup_config_default(airg_setup_config* c) {
  c->strength_alpha = 0.5;
  c->cf = 0;
  c->ddc_enabled = 1;
  c->ddc_fraction = 0.10;
  c->ddc_bins = 1000;
  c->max_loops = 3;
  c->poly_order = 6;
  c->sparsity_order = 1;
  c->drop_coarse = 0.001;
  c->drop_restrict = 0.01;
  c->coarse_size_target = 3000;
  c->coarse_poly_order = 12;
  c->coarse_iterations = 3;
  c->max_levels = 0;
  c->prolongation = 0;
  c->weight_mode = 0;
  c->seed = 0;
  c->fused_smooths = -1;
  c->_pad = 0;
}

void airg_solve_config_default(airg_solve_config* c) {
  c->rtol = 1e-10;
  c->max_iterations = 200;
  c->up_f_smooths = 2;
  c->down_smooths = 0;
  c->coarse_iterations = 3;
  c->collect_timing = 1;
  c->outer = 0;
  c->nddofs = 0;
  c->gmres_restart = 30;
  c->fast = 0;
  c->_pad2 = 0;
}

int airg_ctx_create(int device, airg_ctx** out) {
  return guard([&] {
    need(out, "output handle");
    auto ctx = std::make_unique<airg_ctx>();
    ctx->c.device = device;
    int count = 0;
    CUDA_CHECK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw InvalidArgument("airg_ctx_create: no such CUDA device");
    CUDA_CHECK(cudaSetDevice(device));
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->c.own_stream, cudaStreamNonBlocking));
    ctx->c.stream = ctx->c.own_stream;
    CUDA_CHECK(cudaDeviceGetAttribute(&ctx->c.num_sms, cudaDevAttrMultiProcessorCount, device));
    cudaMemPool_t pool;
    CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = ctx.release();
  });
}

int airg_ctx_destroy(airg_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    bind(ctx->c);
    cudaStreamSynchronize(ctx->c.stream);
    ctx_free_workers(ctx->c);
    if (ctx->c.scratch) cudaFree(ctx->c.scratch);
    if (ctx->c.grid_bar) cudaFree(ctx->c.grid_bar);
    if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.own_stream);
    delete ctx;
  });
}

int airg_ctx_set_stream(airg_ctx* ctx, void* stream) {
  return guard([&] {
    need(ctx, "context");
    ctx->c.stream = stream ? (cudaStream_t)stream : ctx->c.own_stream;
  });
}

int airg_ctx_synchronize(airg_ctx* ctx) {
  return guard([&] {
    need(ctx, "context");
    bind(ctx->c);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_ctx_launch_count(airg_ctx* ctx, uint64_t* out) {
  return guard([&] {
    need(ctx, "context");
    *out = ctx->c.launches;
  });
}

// ---- CSR --------------------------------------------------------------------
int airg_csr_upload(airg_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* rp,
                    const int64_t* ci, const double* v, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output handle");
    bind(ctx->c);
    auto h = std::make_unique<airg_csr>();
    h->c = &ctx->c;
    csr_upload(ctx->c, nrows, ncols, rp, ci, v, h->m);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
    *out = h.release();
  });
}

int airg_csr_info(const airg_csr* a, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  return guard([&] {
    need(a, "matrix");
    if (nrows) *nrows = a->m.n;
    if (ncols) *ncols = a->m.m;
    if (nnz) *nnz = a->m.nnz;
  });
}

int airg_csr_download(airg_ctx* ctx, const airg_csr* a, int64_t* rp, int64_t* ci, double* v) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    csr_download(ctx->c, a->m, rp, ci, v);
  });
}

int airg_csr_device_ptrs(const airg_csr* a, const int32_t** rp, const int32_t** ci,
                         const double** v) {
  return guard([&] {
    need(a, "matrix");
    if (rp) *rp = a->m.rp.p;
    if (ci) *ci = a->m.ci.p;
    if (v) *v = a->m.v.p;
  });
}

int airg_csr_destroy(airg_csr* a) {
  return guard([&] { delete a; });
}

static airg_csr* wrap(Ctx& c, Csr&& m) {
  auto h = new airg_csr;
  h->c = &c;
  h->m = std::move(m);
  return h;
}

int airg_spmv(airg_ctx* ctx, const airg_csr* a, const double* x, double* y) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    if (a->m.n && (!x || !y) && a->m.m) throw InvalidArgument("spmv: dimension mismatch");
    spmv(ctx->c, a->m, x, y);
  });
}

// ---- device buffers for hosts without the CUDA runtime (C / C++ / FFI) -----------
int airg_device_alloc(airg_ctx* ctx, size_t bytes, void** out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output pointer");
    bind(ctx->c);
    *out = nullptr;
    CUDA_CHECK(cudaMallocAsync(out, bytes ? bytes : 16, ctx->c.stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}
int airg_device_free(airg_ctx* ctx, void* p) {
  return guard([&] {
    need(ctx, "context");
    bind(ctx->c);
    if (p) CUDA_CHECK(cudaFreeAsync(p, ctx->c.stream));
  });
}
int airg_memcpy(airg_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t to_device) {
  return guard([&] {
    need(ctx, "context");
    bind(ctx->c);
    if (!bytes) return;
    need(dst, "destination pointer");
    need(src, "source pointer");
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                               ctx->c.stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_spmv_host(airg_ctx* ctx, const airg_csr* a, const double* hx, double* hy) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Ctx& c = ctx->c;
    DBuf<double> dx(c, (size_t)a->m.m), dy(c, (size_t)a->m.n);
    to_device(c, dx.p, hx, (size_t)a->m.m);
    spmv(c, a->m, dx.p, dy.p);
    to_host(c, hy, dy.p, (size_t)a->m.n);
  });
}

int airg_cf_split_host(airg_ctx* ctx, const airg_csr* a, double alpha, int64_t max_loops,
                       uint64_t seed, int32_t weight_mode, int32_t ddc_enabled, double ddc_fraction,
                       int64_t ddc_bins, uint8_t* h_labels, airg_cf_report* rep) {
  int rc = AIRG_OK;
  int rc2 = guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(h_labels, "labels");
    bind(ctx->c);
    DBuf<uint8_t> d(ctx->c, (size_t)std::max(1, a->m.n));
    rc = airg_cf_split(ctx, a, alpha, max_loops, seed, weight_mode, ddc_enabled, ddc_fraction,
                       ddc_bins, d.p, nullptr, rep);
    if (rc == AIRG_OK) to_host(ctx->c, h_labels, d.p, (size_t)a->m.n);
  });
  return rc != AIRG_OK ? rc : rc2;
}

int airg_spgemm(airg_ctx* ctx, const airg_csr* a, const airg_csr* b, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(b, "matrix");
    bind(ctx->c);
    Csr r;
    spgemm(ctx->c, a->m, b->m, r);
    *out = wrap(ctx->c, std::move(r));
  });
}

int airg_drop(airg_ctx* ctx, const airg_csr* a, double tol, int keep_diagonal, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Csr r;
    drop_entries(ctx->c, a->m, tol, keep_diagonal != 0, r);
    *out = wrap(ctx->c, std::move(r));
  });
}

int airg_with_full_diagonal(airg_ctx* ctx, const airg_csr* a, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Csr r;
    with_full_diagonal(ctx->c, a->m, r);
    *out = wrap(ctx->c, std::move(r));
  });
}

// ---- CF splitting -------------------------------------------------------------
int airg_strength(airg_ctx* ctx, const airg_csr* a, double alpha, airg_csr** s_out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Strength g;
    strength(ctx->c, a->m, alpha, g);
    Csr s;
    s.n = s.m = g.n;
    s.nnz = g.nnz;
    s.rp = std::move(g.rp);
    s.ci = std::move(g.ci);
    s.v.alloc(ctx->c, (size_t)g.nnz);
    if (g.nnz) {
      std::vector<double> ones((size_t)g.nnz, 1.0);
      to_device(ctx->c, s.v.p, ones.data(), ones.size());
    }
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
    *s_out = wrap(ctx->c, std::move(s));
  });
}

int airg_pmisr(airg_ctx* ctx, const airg_csr* a, double alpha, int64_t max_loops, uint64_t seed,
               int32_t weight_mode, uint8_t* labels, double* weights) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Strength g;
    strength(ctx->c, a->m, alpha, g);
    pmisr(ctx->c, g, max_loops, seed, weight_mode, labels, weights);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_pmis(airg_ctx* ctx, const airg_csr* a, double alpha, int32_t swap, uint64_t seed, uint8_t* labels) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(labels, "labels");
    bind(ctx->c);
    Strength g;
    strength(ctx->c, a->m, alpha, g);
    pmis(ctx->c, g, swap != 0, seed, labels);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_pmisr_with_weights(airg_ctx* ctx, const airg_csr* s_pattern, int64_t max_loops,
                            const double* weights, uint8_t* labels) {
  return guard([&] {
    need(ctx, "context");
    need(s_pattern, "pattern");
    bind(ctx->c);
    Strength g;
    strength_from_pattern(ctx->c, s_pattern->m, g);
    pmisr_with_weights(ctx->c, g, max_loops, weights, labels);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

namespace {
Csr copy_csr(Ctx& c, const Csr& a) {
  Csr o;
  o.alloc(c, a.n, a.m, a.nnz);
  CUDA_CHECK(cudaMemcpyAsync(o.rp.p, a.rp.p, sizeof(int32_t) * (a.n + 1), cudaMemcpyDeviceToDevice, c.stream));
  if (a.nnz) {
    CUDA_CHECK(cudaMemcpyAsync(o.ci.p, a.ci.p, sizeof(int32_t) * a.nnz, cudaMemcpyDeviceToDevice, c.stream));
    CUDA_CHECK(cudaMemcpyAsync(o.v.p, a.v.p, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, c.stream));
  }
  return o;
}
}  // namespace

int airg_pmisr_pattern(airg_ctx* ctx, const airg_csr* s_pattern, int64_t max_loops, uint64_t seed,
                       int32_t weight_mode, uint8_t* labels, double* weights) {
  return guard([&] {
    need(ctx, "context");
    need(s_pattern, "pattern");
    need(labels, "labels");
    bind(ctx->c);
    Strength g;
    strength_from_pattern(ctx->c, s_pattern->m, g);
    pmisr(ctx->c, g, max_loops, seed, weight_mode, labels, weights);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_pmis_pattern(airg_ctx* ctx, const airg_csr* s_pattern, int32_t swap, uint64_t seed, uint8_t* labels) {
  return guard([&] {
    need(ctx, "context");
    need(s_pattern, "pattern");
    need(labels, "labels");
    bind(ctx->c);
    Strength g;
    strength_from_pattern(ctx->c, s_pattern->m, g);
    pmis(ctx->c, g, swap != 0, seed, labels);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
  });
}

int airg_ddc_block(airg_ctx* ctx, const airg_csr* a_ff, uint8_t* labels, int64_t n, double fraction, int64_t bins,
                   int32_t selection, double direct_alpha, airg_cf_report* rep) {
  return guard([&] {
    need(ctx, "context");
    need(a_ff, "matrix");
    need(labels, "labels");
    bind(ctx->c);
    if (n < 0 || n > INT32_MAX) throw InvalidArgument("ddc: length out of range");
    Ctx& c = ctx->c;
    LabelMap map;
    build_label_map(c, labels, (int32_t)n, map);
    if (a_ff->m.n != map.nf || a_ff->m.m != map.nf) throw InvalidArgument("ddc: a_ff does not match the labels");
    DdcResult d = ddc(c, a_ff->m, map, labels, fraction, bins, selection, direct_alpha, true);
    airg_cf_report r;
    std::memset(&r, 0, sizeof r);
    r.n_f_pre = map.nf;
    r.max_theta = d.max_theta;
    r.alpha_diag = d.alpha_diag;
    r.n_converted = d.converted;
    r.n_f = map.nf - d.converted;
    r.n_c = n - r.n_f;
    if (rep) *rep = r;
  });
}

int airg_hier_from_levels(airg_ctx* ctx, int64_t n_levels, const airg_csr* const* mats,
                          const uint8_t* const* d_labels, const airg_csr* coarse_a, const airg_csr* coarse_inv,
                          int64_t coarse_iterations, airg_hier** out) {
  return guard([&] {
    need(ctx, "context");
    need(coarse_a, "coarse matrix");
    need(coarse_inv, "coarse inverse");
    need(out, "output handle");
    if (n_levels < 0) throw InvalidArgument("hierarchy: negative level count");
    if (n_levels && (!mats || !d_labels)) throw InvalidArgument("hierarchy: null level arrays");
    bind(ctx->c);
    Ctx& c = ctx->c;
    std::vector<HostLevel> lv((size_t)n_levels);
    for (int64_t l = 0; l < n_levels; ++l) {
      const airg_csr* const* m = mats + 7 * l;
      for (int k = 0; k < 7; ++k) need(m[k], "level matrix");
      need(d_labels[l], "level labels");
      lv[l].a = copy_csr(c, m[0]->m);
      lv[l].aff = copy_csr(c, m[1]->m);
      lv[l].afc = copy_csr(c, m[2]->m);
      lv[l].acf = copy_csr(c, m[3]->m);
      lv[l].ffinv = copy_csr(c, m[4]->m);
      lv[l].r = copy_csr(c, m[5]->m);
      lv[l].p = copy_csr(c, m[6]->m);
      lv[l].labels = d_labels[l];
    }
    auto h = std::make_unique<airg_hier>();
    h->c = &c;
    hier_from_levels(c, lv, copy_csr(c, coarse_a->m), copy_csr(c, coarse_inv->m), coarse_iterations, h->h);
    *out = h.release();
  });
}

// AIRG_CF=legacy: the step-by-step split (materialised S, label map, A_ff)
static bool cf_split_legacy() {
  static const bool v = [] {
    const char* e = getenv("AIRG_CF");
    return e && !strcmp(e, "legacy");
  }();
  return v;
}

int airg_cf_split(airg_ctx* ctx, const airg_csr* a, double alpha, int64_t max_loops, uint64_t seed,
                  int32_t weight_mode, int32_t ddc_enabled, double ddc_fraction, int64_t ddc_bins,
                  uint8_t* labels, uint8_t* labels_pre, airg_cf_report* rep) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(labels, "labels");
    bind(ctx->c);
    Ctx& c = ctx->c;
    if (max_loops < 1) throw InvalidArgument("pmisr: max_loops must be >= 1");
    if (weight_mode == 0 && !cf_split_legacy()) {
      const CfFused f = cf_split_fused(c, a->m, alpha, seed, ddc_enabled != 0, ddc_fraction, ddc_bins,
                                       labels, labels_pre);
      airg_cf_report r;
      std::memset(&r, 0, sizeof r);
      r.n_f_pre = f.n_f_pre;
      r.s_nnz = f.s_nnz;
      r.max_theta = f.max_theta;
      r.alpha_diag = f.alpha_diag;
      r.n_converted = f.n_converted;
      r.n_f = r.n_f_pre - r.n_converted;
      r.n_c = a->m.n - r.n_f;
      if (rep) *rep = r;
      return;
    }
    Strength g;
    strength(c, a->m, alpha, g);
    pmisr(c, g, max_loops, seed, weight_mode, labels, nullptr);
    if (labels_pre && a->m.n)
      CUDA_CHECK(cudaMemcpyAsync(labels_pre, labels, a->m.n, cudaMemcpyDeviceToDevice, c.stream));
    LabelMap map;
    build_label_map(c, labels, a->m.n, map);
    airg_cf_report r;
    std::memset(&r, 0, sizeof r);
    r.n_f_pre = map.nf;
    r.s_nnz = g.nnz;
    if (ddc_enabled && map.nf > 0) {
      Blocks blk;
      extract_blocks(c, a->m, map, blk, false);
      DdcResult d = ddc(c, blk.aff, map, labels, ddc_fraction, ddc_bins, 0, 0.0, true);
      r.max_theta = d.max_theta;
      r.alpha_diag = d.alpha_diag;
      r.n_converted = d.converted;
    }
    r.n_f = r.n_f_pre - r.n_converted;
    r.n_c = a->m.n - r.n_f;
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (rep) *rep = r;
  });
}

int airg_cf_split_batch(airg_ctx* ctx, const airg_csr* const* mats, int64_t count, const uint64_t* seeds,
                        double alpha, int64_t max_loops, int32_t ddc_enabled, double ddc_fraction,
                        int64_t ddc_bins, uint8_t* const* labels, airg_cf_report* reps) {
  return guard([&] {
    need(ctx, "context");
    if (count < 0) throw InvalidArgument("cf_split_batch: count must be >= 0");
    if (count == 0) return;
    need(mats, "matrices");
    need(seeds, "seeds");
    need(labels, "labels");
    need(reps, "reports");
    if (max_loops < 1) throw InvalidArgument("pmisr: max_loops must be >= 1");
    for (int64_t i = 0; i < count; ++i) {
      need(mats[i], "matrix");
      if (mats[i]->m.n) need(labels[i], "labels");
    }
    bind(ctx->c);
    Ctx& c = ctx->c;
    DBuf<unsigned long long> u(c, 8 * (size_t)count);
    // every level's counters / histogram / counts / marks in one region,
    // zeroed by one memset before the first split (no zeroing kernel on the
    // chain of each level)
    std::vector<size_t> off((size_t)count + 1, 0);
    for (int64_t i = 0; i < count; ++i)
      off[i + 1] = off[i] + cf_split_zero_bytes(mats[i]->m.n, ddc_enabled != 0, ddc_bins);
    DBuf<uint8_t> zr(c, std::max<size_t>(off[count], 16));
    CUDA_CHECK(cudaMemsetAsync(zr.p, 0, off[count], c.stream));
    CUDA_CHECK(cudaMemsetAsync(u.p, 0, sizeof(unsigned long long) * 8 * count, c.stream));
    for (int64_t i = 0; i < count; ++i)
      cf_split_fused_enqueue(c, mats[i]->m, alpha, seeds[i], ddc_enabled != 0, ddc_fraction, ddc_bins, labels[i],
                             nullptr, u.p + 8 * i, zr.p + off[i]);
    std::vector<unsigned long long> hu(8 * (size_t)count);
    to_host(c, hu.data(), u.p, hu.size());
    for (int64_t i = 0; i < count; ++i) {
      const CfFused f = cf_split_fused_finish(c, hu.data() + 8 * i, ddc_enabled != 0, labels[i]);
      airg_cf_report r;
      std::memset(&r, 0, sizeof r);
      r.n_f_pre = f.n_f_pre;
      r.s_nnz = f.s_nnz;
      r.max_theta = f.max_theta;
      r.alpha_diag = f.alpha_diag;
      r.n_converted = f.n_converted;
      r.n_f = r.n_f_pre - r.n_converted;
      r.n_c = mats[i]->m.n - r.n_f;
      reps[i] = r;
    }
  });
}

int airg_ddc(airg_ctx* ctx, const airg_csr* a, uint8_t* labels, double fraction, int64_t bins,
             int32_t selection, double direct_alpha, airg_cf_report* rep) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Ctx& c = ctx->c;
    LabelMap map;
    build_label_map(c, labels, a->m.n, map);
    Blocks blk;
    extract_blocks(c, a->m, map, blk, false);
    DdcResult d = ddc(c, blk.aff, map, labels, fraction, bins, selection, direct_alpha, true);
    airg_cf_report r;
    std::memset(&r, 0, sizeof r);
    r.n_f_pre = map.nf;
    r.max_theta = d.max_theta;
    r.alpha_diag = d.alpha_diag;
    r.n_converted = d.converted;
    r.n_f = map.nf - d.converted;
    r.n_c = a->m.n - r.n_f;
    if (rep) *rep = r;
  });
}

int airg_extract_blocks(airg_ctx* ctx, const airg_csr* a, const uint8_t* labels, airg_csr** aff,
                        airg_csr** afc, airg_csr** acf) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    if (a->m.n != a->m.m) throw InvalidArgument("extract_blocks: label length mismatch");
    LabelMap map;
    build_label_map(ctx->c, labels, a->m.n, map);
    Blocks blk;
    extract_blocks(ctx->c, a->m, map, blk, false);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
    if (aff) *aff = wrap(ctx->c, std::move(blk.aff));
    if (afc) *afc = wrap(ctx->c, std::move(blk.afc));
    if (acf) *acf = wrap(ctx->c, std::move(blk.acf));
  });
}

// dominance_report (coarsening.cpp:219-250) of an A_ff block
int airg_dominance_report(airg_ctx* ctx, const airg_csr* a_ff, int64_t bins, double* d_theta,
                          int64_t* h_hist, double* max_theta) {
  return guard([&] {
    need(ctx, "context");
    need(a_ff, "matrix");
    bind(ctx->c);
    const double mx = dominance_report(ctx->c, a_ff->m, bins, d_theta, h_hist);
    if (max_theta) *max_theta = mx;
  });
}

// build_label_map (sparse.cpp:270-290): F-then-C sub-indexing, host outputs
int airg_build_label_map(airg_ctx* ctx, const uint8_t* d_labels, int64_t n, int64_t* h_fine_to_sub,
                         int64_t* h_f_to_fine, int64_t* h_c_to_fine, int64_t* n_f) {
  return guard([&] {
    need(ctx, "context");
    bind(ctx->c);
    if (n < 0 || n > INT32_MAX) throw InvalidArgument("build_label_map: length out of range");
    LabelMap map;
    build_label_map(ctx->c, d_labels, (int32_t)n, map);
    auto out = [&](const DBuf<int32_t>& d, int64_t len, int64_t* h) {
      if (!h || len == 0) return;
      std::vector<int32_t> t((size_t)len);
      to_host(ctx->c, t.data(), d.p, t.size());
      for (int64_t k = 0; k < len; ++k) h[k] = t[(size_t)k];
    };
    out(map.fine_to_sub, n, h_fine_to_sub);
    out(map.f_to_fine, map.nf, h_f_to_fine);
    out(map.c_to_fine, map.nc, h_c_to_fine);
    if (n_f) *n_f = map.nf;
  });
}

// ---- transfer operators (air.hpp:96-116) ------------------------------------------
int airg_build_restriction(airg_ctx* ctx, const airg_csr* a_cf, const airg_csr* aff_inv, double drop_restrict,
                           const uint8_t* d_labels, int64_t n, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a_cf, "matrix");
    need(aff_inv, "matrix");
    need(out, "output handle");
    bind(ctx->c);
    if (n < 0 || n > INT32_MAX) throw InvalidArgument("build_restriction: length out of range");
    LabelMap map;
    build_label_map(ctx->c, d_labels, (int32_t)n, map);
    if (a_cf->m.n != map.nc || a_cf->m.m != map.nf || aff_inv->m.n != map.nf || aff_inv->m.m != map.nf)
      throw InvalidArgument("build_restriction: block shapes do not match the label map");
    Csr r;
    build_restriction(ctx->c, a_cf->m, aff_inv->m, drop_restrict, map, r);
    *out = wrap(ctx->c, std::move(r));
  });
}

// one-point prolongation from the strength pattern S (airg_strength) and A
int airg_build_prolongation(airg_ctx* ctx, const airg_csr* a, const airg_csr* s, const uint8_t* d_labels,
                            airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(s, "strength pattern");
    need(out, "output handle");
    bind(ctx->c);
    if (s->m.n != a->m.n || a->m.n != a->m.m) throw InvalidArgument("build_prolongation: shape mismatch");
    LabelMap map;
    build_label_map(ctx->c, d_labels, a->m.n, map);
    Strength g;
    strength_from_pattern(ctx->c, s->m, g);
    DBuf<int32_t> pmap;
    Csr p;
    build_prolongation(ctx->c, map, g, a->m, pmap, p);
    *out = wrap(ctx->c, std::move(p));
  });
}

// coarse_matrix (air.cpp:268-271): drop_entries(R (A P), drop_coarse)
int airg_coarse_matrix(airg_ctx* ctx, const airg_csr* r, const airg_csr* a, const airg_csr* p, double drop_coarse,
                       airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(r, "matrix");
    need(a, "matrix");
    need(p, "matrix");
    need(out, "output handle");
    bind(ctx->c);
    if (a->m.m != p->m.n || r->m.m != a->m.n) throw InvalidArgument("spgemm: dimension mismatch");  // sparse.cpp:206
    Csr ap, rap, res;
    spgemm(ctx->c, a->m, p->m, ap);
    spgemm(ctx->c, r->m, ap, rap);
    drop_entries(ctx->c, rap, drop_coarse, true, res);
    *out = wrap(ctx->c, std::move(res));
  });
}

// ---- polynomials ----------------------------------------------------------------
// apply_polynomial (gmres_poly.cpp:173-195): d_y = q(A) d_b, Horner
int airg_apply_polynomial(airg_ctx* ctx, const airg_csr* a, const double* coeffs, int64_t ncoeffs,
                          int64_t effective_order, const double* d_b, double* d_y) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(coeffs, "coefficients");
    bind(ctx->c);
    apply_polynomial(ctx->c, const_cast<airg_csr*>(a)->m, coeffs, ncoeffs, effective_order, d_b, d_y);  // row-layout cache only
  });
}
int airg_poly_coefficients(airg_ctx* ctx, const airg_csr* a, int64_t m, uint64_t seed,
                           double* coeffs, int64_t* eff) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    PolyFit f = poly_coefficients(ctx->c, a->m, m, seed);
    std::memcpy(coeffs, f.coeffs.data(), sizeof(double) * f.coeffs.size());
    if (eff) *eff = f.effective_order;
  });
}

int airg_poly_assemble(airg_ctx* ctx, const airg_csr* a, const double* coeffs, int64_t ncoeffs,
                       int64_t eff, int64_t sparsity_order, airg_csr** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    bind(ctx->c);
    Csr r;
    poly_assemble(ctx->c, a->m, coeffs, ncoeffs, eff, sparsity_order, r);
    CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
    *out = wrap(ctx->c, std::move(r));
  });
}

// ---- setup --------------------------------------------------------------------------
namespace {
int setup_impl(airg_ctx* ctx, const airg_csr* a, const airg_setup_config* cfg, const airg_injection* inj,
               airg_hier** out, const RowSplit* rs) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(cfg, "config");
    need(out, "output handle");
    bind(ctx->c);
    auto h = std::make_unique<airg_hier>();
    h->c = &ctx->c;
    std::unique_ptr<Injection> in;
    if (inj) {
      in = std::make_unique<Injection>();
      in->n_levels = inj->n_levels;
      for (int64_t l = 0; l < inj->n_levels; ++l) {
        in->level_coeffs.emplace_back(inj->level_coeffs + l * inj->stride,
                                      inj->level_coeffs + l * inj->stride + cfg->poly_order + 1);
        in->level_eff.push_back(inj->level_eff_order[l]);
      }
      in->coarse_coeffs.assign(inj->coarse_coeffs, inj->coarse_coeffs + cfg->coarse_poly_order + 1);
      in->coarse_eff = inj->coarse_eff_order;
    }
    setup(ctx->c, a->m, *cfg, in.get(), h->h, rs);
    *out = h.release();
  });
}
}  // namespace

int airg_setup(airg_ctx* ctx, const airg_csr* a, const airg_setup_config* cfg,
               const airg_injection* inj, airg_hier** out) {
  return setup_impl(ctx, a, cfg, inj, out, nullptr);
}

int airg_dist_setup(airg_ctx* ctx, const airg_csr* a, const airg_setup_config* cfg,
                    const airg_injection* inj, int32_t nranks, int32_t rank, void* nccl_comm,
                    airg_hier** out) {
  if (nranks < 1 || rank >= nranks) {
    g_err = "dist_setup: rank out of range";
    return AIRG_EINVAL;
  }
  if (rank >= 0 && nranks > 1 && !nccl_comm) {
    g_err = "dist_setup: a communicator is needed per rank";
    return AIRG_EINVAL;
  }
  RowSplit rs;
  rs.P = nranks;
  rs.me = rank;
  rs.comm = (ncclComm_t)nccl_comm;
  return setup_impl(ctx, a, cfg, inj, out, &rs);
}

int airg_hier_info_get(const airg_hier* hp, airg_hier_info* info) {
  return guard([&] {
    need(hp, "hierarchy");
    const Hier& h = hp->h;
    std::memset(info, 0, sizeof *info);
    info->n_levels = (int64_t)h.levels.size();
    info->coarse_n = h.coarse_a.n;
    info->coarse_nnz = h.coarse_a.nnz;
    info->coarse_inv_nnz = h.coarse_inv.nnz;
    info->coarse_effective_order = h.coarse_eff;
    info->coarse_attempts = h.coarse_attempts;
    info->coarse_growth = h.coarse_growth;
    for (size_t k = 0; k < h.coarse_coeffs.size() && k < 32; ++k)
      info->coarse_coefficients[k] = h.coarse_coeffs[k];
    info->grid_complexity = h.grid_c;
    info->operator_complexity = h.op_c;
    info->storage_complexity = h.store_c;
  });
}

int airg_hier_level_info(const airg_hier* hp, int64_t l, airg_level_info* info) {
  return guard([&] {
    need(hp, "hierarchy");
    const Hier& h = hp->h;
    if (l < 0 || l >= (int64_t)h.levels.size()) throw InvalidArgument("level out of range");
    const Level& L = h.levels[l];
    std::memset(info, 0, sizeof *info);
    info->n = L.a.n;
    info->nnz = L.a.nnz;
    info->n_f = L.map.nf;
    info->n_c = L.map.nc;
    info->n_f_pre = L.n_f_pre;
    info->ddc_converted = L.n_converted;
    info->nnz_ff = L.aff.nnz;
    info->nnz_fc = L.afc.nnz;
    info->nnz_cf = L.acf.nnz;
    info->nnz_ffinv = L.ffinv.nnz;
    info->nnz_r = L.r.nnz;
    info->nnz_p = L.p.nnz;
    info->max_theta_pre = L.max_theta_pre;
    info->alpha_diag = L.alpha_diag;
    info->max_theta_post = L.max_theta_post;
    info->smoother_growth = L.growth;
    info->poly_attempts = L.attempts;
    info->effective_order = L.eff;
    for (size_t k = 0; k < L.coeffs.size() && k < 32; ++k) info->coefficients[k] = L.coeffs[k];
  });
}

int airg_hier_matrix(const airg_hier* hp, int64_t l, int32_t which, const airg_csr** out) {
  return guard([&] {
    need(hp, "hierarchy");
    airg_hier* h = const_cast<airg_hier*>(hp);
    const int64_t nl = (int64_t)h->h.levels.size();
    const Csr* m = nullptr;
    if (l == nl) {
      if (which == 0) m = &h->h.coarse_a;
      else if (which == 4) m = &h->h.coarse_inv;
      else if (which == 9 && h->h.coarse_composed) m = &h->h.coarse_e;
      else throw InvalidArgument("coarse level has only A (0), inverse (4) and a composed solve (9)");
    } else {
      if (l < 0 || l > nl) throw InvalidArgument("level out of range");
      const Level& L = h->h.levels[l];
      const Csr* ms[11] = {&L.a, &L.aff, &L.afc, &L.acf, &L.ffinv, &L.r, &L.p, &L.afp, &L.fw, &L.fk, &L.dsc};
      if (which < 0 || which > 10) throw InvalidArgument("bad matrix selector");
      if (which >= 7 && h->h.fused_smooths < 0)
        throw InvalidArgument("fast V-cycle operators not built (setup fused_smooths >= 0 or a fast solve)");
      if (which >= 9 && !L.one_pass) throw InvalidArgument("level has no one-pass ascent operators");
      m = ms[which];
    }
    // borrowed view: a handle whose Csr aliases the hierarchy's buffers
    auto v = std::make_unique<airg_csr>();
    v->c = h->c;
    v->m.n = m->n;
    v->m.m = m->m;
    v->m.nnz = m->nnz;
    v->m.rp.p = m->rp.p;
    v->m.ci.p = m->ci.p;
    v->m.v.p = m->v.p;
    *out = v.get();
    h->views.push_back(std::move(v));
  });
}

int airg_hier_labels(airg_ctx* ctx, const airg_hier* hp, int64_t l, uint8_t* h_labels) {
  return guard([&] {
    need(ctx, "context");
    need(hp, "hierarchy");
    bind(ctx->c);
    const Hier& h = hp->h;
    if (l < 0 || l >= (int64_t)h.levels.size()) throw InvalidArgument("level out of range");
    to_host(ctx->c, h_labels, h.levels[l].map.label.p, (size_t)h.levels[l].map.n);
  });
}

int airg_hier_destroy(airg_hier* h) {
  return guard([&] {
    if (!h) return;
    for (auto& v : h->views) {  // views alias; do not free their buffers
      v->m.rp.p = nullptr;
      v->m.ci.p = nullptr;
      v->m.v.p = nullptr;
    }
    if (h->c) bind(*h->c);
    delete h;
  });
}

// ---- solve --------------------------------------------------------------------------
int airg_f_smooth(airg_ctx* ctx, const airg_hier* hp, int64_t level, const double* d_b, double* d_x) {
  return guard([&] {
    need(ctx, "context");
    need(hp, "hierarchy");
    bind(ctx->c);
    f_smooth_level(ctx->c, const_cast<airg_hier*>(hp)->h, level, d_b, d_x);
  });
}

int airg_vcycle(airg_ctx* ctx, const airg_hier* hp, const airg_solve_config* cfg, const double* b,
                double* x) {
  return guard([&] {
    need(ctx, "context");
    need(hp, "hierarchy");
    need(cfg, "config");
    bind(ctx->c);
    vcycle(ctx->c, const_cast<airg_hier*>(hp)->h, *cfg, b, x);
  });
}

int airg_solve(airg_ctx* ctx, const airg_hier* hp, const airg_solve_config* cfg, const double* b,
               double* x, airg_solve_stats* st, double* hist, int64_t cap) {
  return guard([&] {
    need(ctx, "context");
    need(hp, "hierarchy");
    need(cfg, "config");
    bind(ctx->c);
    std::vector<double> h;
    airg_solve_stats s;
    solve(ctx->c, const_cast<airg_hier*>(hp)->h, *cfg, b, x, s, h);
    if (hist)
      for (int64_t k = 0; k < cap && k < (int64_t)h.size(); ++k) hist[k] = h[k];
    if (st) *st = s;
  });
}

int airg_solve_host(airg_ctx* ctx, const airg_hier* hp, const airg_solve_config* cfg,
                    const double* h_b, double* h_x, airg_solve_stats* st, double* hist, int64_t cap) {
  return guard([&] {
    need(ctx, "context");
    need(hp, "hierarchy");
    need(cfg, "config");
    bind(ctx->c);
    Ctx& c = ctx->c;
    Hier& h = const_cast<airg_hier*>(hp)->h;
    const int n = h.top_n();
    DBuf<double> db(c, (size_t)n), dx(c, (size_t)n);
    CUDA_CHECK(cudaMemcpyAsync(db.p, h_b, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
    std::vector<double> hv;
    airg_solve_stats s;
    solve(c, h, *cfg, db.p, dx.p, s, hv);
    CUDA_CHECK(cudaMemcpyAsync(h_x, dx.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (hist)
      for (int64_t k = 0; k < cap && k < (int64_t)hv.size(); ++k) hist[k] = hv[k];
    if (st) *st = s;
  });
}

// ---- multi-GPU ----------------------------------------------------------------------
struct airg_dist {
  Ctx* c = nullptr;
  DHier d;
};

int airg_nccl_unique_id(void* id) {
  return guard([&] {
    need(id, "id buffer");
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) throw CudaError("ncclGetUniqueId failed");
    static_assert(sizeof(u) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id, &u, sizeof u);
  });
}

int airg_nccl_comm_create(int nranks, int rank, const void* id, void** comm) {
  return guard([&] {
    need(id, "id");
    need(comm, "comm out");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t cm;
    const ncclResult_t r = ncclCommInitRank(&cm, nranks, u, rank);
    if (r != ncclSuccess) throw CudaError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *comm = cm;
  });
}

int airg_nccl_comm_destroy(void* comm) {
  return guard([&] {
    if (comm) ncclCommDestroy((ncclComm_t)comm);
  });
}

int airg_dist_create(airg_ctx* ctx, const airg_hier* h, int32_t nranks, int32_t rank, void* comm,
                     double threshold, const int64_t* starts, airg_dist** out) {
  return guard([&] {
    need(ctx, "context");
    need(h, "hierarchy");
    need(out, "output handle");
    bind(ctx->c);
    auto d = std::make_unique<airg_dist>();
    d->c = &ctx->c;
    dist_create(ctx->c, const_cast<airg_hier*>(h)->h, nranks, rank, (ncclComm_t)comm, threshold, starts,
                d->d);
    *out = d.release();
  });
}

int airg_dist_setup_owned(airg_ctx* ctx, const airg_csr* a, const int64_t* starts, const airg_setup_config* cfg,
                          const airg_injection* inj, int32_t nranks, int32_t rank, void* comm, double threshold,
                          airg_dist** out) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(starts, "starts");
    need(cfg, "config");
    need(out, "output handle");
    bind(ctx->c);
    if (nranks < 1 || rank >= nranks) throw InvalidArgument("dist: rank out of range");
    if (rank >= 0 && nranks > 1 && !comm) throw InvalidArgument("dist: a communicator is needed per rank");
    const std::vector<int64_t> s(starts, starts + nranks + 1);
    for (int r = 0; r < nranks; ++r)
      if (s[r + 1] < s[r]) throw InvalidArgument("dist: slab starts must be non-decreasing");
    if (s[0] != 0) throw InvalidArgument("dist: slab starts must begin at 0");
    std::unique_ptr<Injection> in;
    if (inj) {
      in = std::make_unique<Injection>();
      in->n_levels = inj->n_levels;
      for (int64_t l = 0; l < inj->n_levels; ++l) {
        in->level_coeffs.emplace_back(inj->level_coeffs + l * inj->stride,
                                      inj->level_coeffs + l * inj->stride + cfg->poly_order + 1);
        in->level_eff.push_back(inj->level_eff_order[l]);
      }
      in->coarse_coeffs.assign(inj->coarse_coeffs, inj->coarse_coeffs + cfg->coarse_poly_order + 1);
      in->coarse_eff = inj->coarse_eff_order;
    }
    std::vector<Csr> rows(nranks);
    if (rank < 0) {  // emulation: the whole operator, cut into the slabs here
      if (a->m.n != s[nranks] || a->m.m != s[nranks]) throw InvalidArgument("dist: slab starts must cover the matrix");
      for (int r = 0; r < nranks; ++r) slice(ctx->c, a->m, s[r], s[r + 1], rows[r]);
    } else {
      if (a->m.n != s[rank + 1] - s[rank]) throw InvalidArgument("dist: local rows do not match the slab starts");
      csr_copy(ctx->c, a->m, rows[rank]);
    }
    auto d = std::make_unique<airg_dist>();
    d->c = &ctx->c;
    dist_setup_owned(ctx->c, rows, s, *cfg, in.get(), nranks, rank, (ncclComm_t)comm, threshold, d->d);
    *out = d.release();
  });
}

int airg_dist_fused_nnz(const airg_dist* dp, int64_t level, int64_t* nnz_afp, int64_t* nnz_w) {
  return guard([&] {
    need(dp, "dist");
    need(nnz_afp, "output");
    need(nnz_w, "output");
    const DHier& d = dp->d;
    if (level < 0 || level >= (int64_t)d.lv.size()) throw InvalidArgument("level out of range");
    if (d.fused_smooths < 0) throw InvalidArgument("dist: no fast V-cycle operators (setup fused_smooths >= 0)");
    *nnz_afp = d.lv[(size_t)level].nnz_afp;
    *nnz_w = d.lv[(size_t)level].nnz_w;
  });
}

int airg_dist_coarse_e_nnz(const airg_dist* dp, int64_t* nnz) {
  return guard([&] {
    need(dp, "dist");
    need(nnz, "output");
    const DHier& d = dp->d;
    if (!d.coarse_e_ok) {
      *nnz = -1;
      return;
    }
    int64_t t = 0;
    for (int r = 0; r < d.P && r < (int)d.rk.size(); ++r)
      if (d.mine(r)) t += d.rk[r].ACE.nnz;
    *nnz = t;
  });
}

int airg_dist_report(const airg_dist* dp, int64_t level, airg_level_info* info, int64_t* n_levels) {
  return guard([&] {
    need(dp, "dist");
    const DHier& d = dp->d;
    if (n_levels) *n_levels = (int64_t)d.lv.size();
    if (!info) return;
    if (!d.owned) throw InvalidArgument("dist: setup reports exist for the owned setup only");
    if (level < 0 || level >= (int64_t)d.summary.size()) throw InvalidArgument("level out of range");
    const DHier::Summary& S = d.summary[level];
    std::memset(info, 0, sizeof *info);
    info->n = S.n;
    info->nnz = S.nnz;
    info->n_f = S.nf;
    info->n_c = S.nc;
    info->n_f_pre = S.n_f_pre;
    info->ddc_converted = S.n_converted;
    info->nnz_ff = S.nnz_ff;
    info->nnz_fc = S.nnz_fc;
    info->nnz_cf = S.nnz_cf;
    info->nnz_ffinv = S.nnz_ffinv;
    info->nnz_r = S.nnz_r;
    info->nnz_p = S.nnz_p;
    info->max_theta_pre = S.max_theta_pre;
    info->alpha_diag = S.alpha_diag;
    info->max_theta_post = S.max_theta_post;
    info->smoother_growth = S.growth;
    info->poly_attempts = S.attempts;
    info->effective_order = S.eff;
    for (size_t k = 0; k < S.coeffs.size() && k < 32; ++k) info->coefficients[k] = S.coeffs[k];
  });
}

int airg_dist_setup_times(const airg_dist* dp, double* setup_ms, double* cf_split_ms) {
  return guard([&] {
    need(dp, "dist");
    if (setup_ms) *setup_ms = dp->d.setup_ms;
    if (cf_split_ms) *cf_split_ms = dp->d.cf_ms;
  });
}

int airg_dist_solve(airg_ctx* ctx, airg_dist* d, const airg_solve_config* cfg, const double* b,
                    double* x, airg_solve_stats* st, double* hist, int64_t cap) {
  return guard([&] {
    need(ctx, "context");
    need(d, "dist");
    need(cfg, "config");
    bind(ctx->c);
    std::vector<double> hv;
    airg_solve_stats s;
    dist_solve(ctx->c, d->d, *cfg, b, x, s, hv);
    if (hist)
      for (int64_t k = 0; k < cap && k < (int64_t)hv.size(); ++k) hist[k] = hv[k];
    if (st) *st = s;
  });
}

int airg_dist_halo_bytes(const airg_dist* dp, const airg_solve_config* cfg, int64_t* vcycle_bytes,
                         int64_t* spmv_bytes) {
  return guard([&] {
    need(dp, "dist");
    need(cfg, "config");
    int64_t v = 0, s = 0;
    dist_halo_bytes(dp->d, *cfg, v, s);
    if (vcycle_bytes) *vcycle_bytes = v;
    if (spmv_bytes) *spmv_bytes = s;
  });
}

int airg_dist_rank_bytes(const airg_dist* dp, int32_t rank, int64_t* bytes) {
  return guard([&] {
    need(dp, "dist");
    need(bytes, "bytes");
    const DHier& d = dp->d;
    if (rank < 0 || rank >= d.P) throw InvalidArgument("dist: rank out of range");
    if (!d.mine(rank)) throw InvalidArgument("dist: rank is not held by this process");
    auto csr = [](const Csr& m) {
      return (int64_t)(m.rp.n * sizeof(int32_t) + m.ci.n * sizeof(int32_t) + m.v.n * sizeof(double));
    };
    auto vec = [&](const DVec& V) {
      return rank < (int)V.rk.size() ? (int64_t)(V.rk[rank].buf.n * sizeof(double)) : (int64_t)0;
    };
    int64_t b = 0;
    for (const DLevel& D : d.lv) {
      if (rank < (int)D.rk.size()) {
        const DLevel::Rank& R = D.rk[rank];
        b += csr(R.R) + csr(R.AF) + csr(R.AFFG) + csr(R.FINV);
        b += (int64_t)((R.pmap.n + R.f2f.n) * sizeof(int32_t) + R.sc.n * sizeof(double));
      }
      b += vec(D.B) + vec(D.X) + vec(D.RF);
    }
    if (rank < (int)d.rk.size()) {
      const DHier::Rank& T = d.rk[rank];
      b += csr(T.A0) + csr(T.AC) + csr(T.ACI) + (int64_t)(T.rhs.n * sizeof(double));
    }
    b += vec(d.CB) + vec(d.CX) + vec(d.CR) + vec(d.XS);
    *bytes = b;
  });
}

int airg_dist_level_share(const airg_dist* dp, int64_t l, double* share_before, double* share_after) {
  return guard([&] {
    need(dp, "dist");
    const DHier& d = dp->d;
    if (l < 0 || l >= (int64_t)d.lv.size()) throw InvalidArgument("level out of range");
    if (share_before) *share_before = d.lv[l].share_before;
    if (share_after) *share_after = d.lv[l].share_after;
  });
}

int airg_dist_level_info(const airg_dist* dp, int64_t l, int32_t* active, double* rb, double* ra,
                         int32_t* trig, int64_t* halo, int64_t* starts) {
  return guard([&] {
    need(dp, "dist");
    const DHier& d = dp->d;
    if (l < 0 || l > (int64_t)d.lv.size()) throw InvalidArgument("level out of range");
    if (l == (int64_t)d.lv.size()) {  // coarsest: gathered
      if (active) *active = 1;
      if (rb) *rb = INFINITY;
      if (ra) *ra = INFINITY;
      if (trig) *trig = 0;
      int64_t hs = 0;
      for (const auto& R : d.CX.rk) hs += R.nhalo;
      if (halo) *halo = hs;
      if (starts) std::memcpy(starts, d.cpart.s.data(), sizeof(int64_t) * d.cpart.s.size());
      return;
    }
    const DLevel& D = d.lv[l];
    if (active) *active = D.active;
    if (rb) *rb = D.ratio_before;
    if (ra) *ra = D.ratio_after;
    if (trig) *trig = D.triggered;
    int64_t hs = 0;
    for (const auto& R : D.X.rk) hs += R.nhalo;
    if (halo) *halo = hs;
    if (starts) std::memcpy(starts, D.fine.s.data(), sizeof(int64_t) * D.fine.s.size());
  });
}

int airg_dist_cf_split(airg_ctx* ctx, const airg_csr* a, int32_t nranks, int32_t rank, void* comm,
                       const int64_t* starts, double alpha, int64_t max_loops, uint64_t seed,
                       int32_t ddc_enabled, double fraction, int64_t bins, uint8_t* labels,
                       airg_cf_report* rep) {
  return guard([&] {
    need(ctx, "context");
    need(a, "matrix");
    need(starts, "starts");
    need(labels, "labels");
    bind(ctx->c);
    if (nranks < 1 || rank >= nranks) throw InvalidArgument("dist: rank out of range");
    if (rank >= 0 && nranks > 1 && !comm) throw InvalidArgument("dist: a communicator is needed per rank");
    CfReport r;
    dist_cf_split(ctx->c, a->m, nranks, rank, (ncclComm_t)comm,
                  std::vector<int64_t>(starts, starts + nranks + 1), alpha, max_loops, seed,
                  ddc_enabled != 0, fraction, bins, labels, r);
    if (rep) {
      std::memset(rep, 0, sizeof *rep);
      rep->n_f_pre = r.n_f_pre;
      rep->n_f = r.n_f;
      rep->n_c = a->m.n - r.n_f;
      rep->n_converted = r.n_converted;
      rep->max_theta = r.max_theta;
      rep->alpha_diag = r.alpha_diag;
      rep->s_nnz = r.s_nnz;
    }
  });
}

struct airg_mm {
  MmHost m;
};

int airg_mm_read(const char* path, airg_mm** out) {
  return guard([&] {
    need(path, "path");
    need(out, "output handle");
    auto h = std::make_unique<airg_mm>();
    mm_read(path, h->m);
    *out = h.release();
  });
}

int airg_mm_dims(const airg_mm* h, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  return guard([&] {
    need(h, "matrix market handle");
    if (nrows) *nrows = h->m.n;
    if (ncols) *ncols = h->m.m;
    if (nnz) *nnz = (int64_t)h->m.ci.size();
  });
}

int airg_mm_copy(const airg_mm* h, int64_t* rp, int64_t* ci, double* v) {
  return guard([&] {
    need(h, "matrix market handle");
    if (rp) std::memcpy(rp, h->m.rp.data(), sizeof(int64_t) * h->m.rp.size());
    if (ci && !h->m.ci.empty()) std::memcpy(ci, h->m.ci.data(), sizeof(int64_t) * h->m.ci.size());
    if (v && !h->m.v.empty()) std::memcpy(v, h->m.v.data(), sizeof(double) * h->m.v.size());
  });
}

int airg_mm_free(airg_mm* h) {
  delete h;
  return AIRG_OK;
}

int airg_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                  const double* v) {
  return guard([&] {
    need(path, "path");
    if (nrows < 0 || ncols < 0) throw InvalidArgument("matrix market: negative dimensions");
    if (nrows > 0) need(rp, "row offsets");
    mm_write(path, nrows, ncols, rp, ci, v);
  });
}

int airg_dist_transport(const airg_dist* dp, int32_t* transport) {
  return guard([&] {
    need(dp, "dist");
    need(transport, "transport");
    const DHier& d = dp->d;
    *transport = d.p2p.on ? 2 : (d.me >= 0 && d.P > 1 ? 1 : 0);
  });
}

int airg_dist_destroy(airg_dist* d) {
  return guard([&] {
    if (!d) return;
    if (d->c) bind(*d->c);
    delete d;
  });
}

int airg_dist_plan_host(int32_t nranks, const int64_t* starts, int32_t rank, const int64_t* cols,
                        int64_t ncols, int64_t* halo_out, int64_t cap, int64_t* n_halo,
                        int64_t* recv_counts) {
  return guard([&] {
    need(starts, "starts");
    if (rank < 0 || rank >= nranks) throw InvalidArgument("dist: rank out of range");
    std::vector<int64_t> s(starts, starts + nranks + 1), halo, rc;
    halo_plan_host(s, rank, cols, ncols, halo, rc);
    if (n_halo) *n_halo = (int64_t)halo.size();
    if (halo_out)
      for (int64_t k = 0; k < cap && k < (int64_t)halo.size(); ++k) halo_out[k] = halo[k];
    if (recv_counts)
      for (int q = 0; q < nranks; ++q) recv_counts[q] = rc[q];
  });
}

int airg_p2p_push_plan_host(int32_t nranks, const int64_t* starts, int32_t sender, const int64_t* recv_halo,
                            int64_t n_recv_halo, int32_t receiver, int32_t* src_idx, int64_t* dst_pos,
                            int64_t cap, int64_t* n_push) {
  return guard([&] {
    need(starts, "starts");
    if (sender < 0 || sender >= nranks || receiver < 0 || receiver >= nranks)
      throw InvalidArgument("dist: rank out of range");
    std::vector<int64_t> halo(recv_halo, recv_halo + n_recv_halo);
    const int64_t recv_own = starts[receiver + 1] - starts[receiver];
    int64_t recv_off = 0;  // the receiver's halo entries owned by lower ranks come first
    for (int64_t g : halo)
      if (g < starts[sender]) ++recv_off;
    std::vector<int32_t> si;
    std::vector<int64_t> pos;
    p2p_push_plan(halo, recv_own, recv_off, starts[sender], starts[sender + 1] - starts[sender], si, pos);
    if (n_push) *n_push = (int64_t)si.size();
    for (int64_t k = 0; k < cap && k < (int64_t)si.size(); ++k) {
      if (src_idx) src_idx[k] = si[k];
      if (dst_pos) dst_pos[k] = pos[k];
    }
  });
}

}  // extern "C"
