/* oracle/airg_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * A plain-C restatement of the reference AIRG hot path
 * (/root/reference/proj/src/{sparse,coarsening,gmres_poly,air,solve}.cpp),
 * used by tests/ (as the parity checker on the GPU box, where
 * /root/reference does not exist), by __graft_entry__.smoke() and by
 * bench.py's cpu_baseline / reference-arm fallback. It is never linked into
 * the product.
 *
 * Every function cites the reference lines it restates and keeps the
 * reference's operation order (sequential row sums in column order, no FMA:
 * build with -ffp-contract=off), so results are bit-identical to the
 * reference build oracle/_ref. The polynomial coefficients follow
 * gmres_poly.cpp:63-171 in x87 long double with the Householder QR and
 * complete-orthogonal-decomposition algorithms of oracle/shim/Eigen/Dense
 * (the reference needs Eigen there, which is absent from this image:
 * against real Eigen the coefficients are "parity unpinned", against the
 * reference's own known-answer tests they are pinned).
 *
 * The outer GMRES (orc_solve with outer = 1) is NOT in the reference
 * (Richardson only, solve.cpp:167-259); it is composed from the restated
 * vcycle() and spmv() exactly as the GPU implements it.
 */
#define _GNU_SOURCE
#include "airg_oracle.h"

#include <float.h>
#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef orc_csr csr;

/* ------------------------------------------------------------------------ */
/* errors: longjmp to the API boundary (leaks on the error path are fine
 * for test infrastructure). */
static __thread char g_err[4096];
static __thread jmp_buf* g_jb;

static void fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  longjmp(*g_jb, -code);
}
#define EINV(...) fail(1, __VA_ARGS__)
#define ERUN(...) fail(2, __VA_ARGS__)

#define API_BEGIN                 \
  jmp_buf jb__;                   \
  jmp_buf* prev__ = g_jb;         \
  int rc__ = setjmp(jb__);        \
  if (rc__ != 0) {                \
    g_jb = prev__;                \
    return rc__;                  \
  }                               \
  g_jb = &jb__;
#define API_END \
  g_jb = prev__; \
  return AIRG_OK;

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) fail(4, "out of memory");
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) fail(4, "out of memory");
  return p;
}

int orc_last_error(char* buf, size_t len) {
  if (buf && len) {
    strncpy(buf, g_err, len - 1);
    buf[len - 1] = 0;
  }
  return (int)strlen(g_err);
}

/* ------------------------------------------------------------------------ */
/* rng.hpp:13-39 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static uint64_t mix(uint64_t seed, uint64_t key) { return splitmix64(seed ^ splitmix64(key)); }
static double uniform01(uint64_t seed, uint64_t index) {
  return (double)(mix(seed, index) >> 11) * 0x1.0p-53;
}
static double standard_normal(uint64_t seed, uint64_t index) {
  const double u1 = (double)((mix(seed, 2 * index) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(mix(seed, 2 * index + 1) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}
#define kStreamWeights 0x57454947ull
#define kStreamPolyRhs 0x504f4c59ull

/* ------------------------------------------------------------------------ */
/* CSR value type, sparse.hpp:33-94 / sparse.cpp:18-46 */
static csr* csr_new(int64_t n, int64_t m, int64_t nnz) {
  csr* a = (csr*)xcalloc(1, sizeof(csr));
  a->n = n;
  a->m = m;
  a->rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
  a->ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)nnz);
  a->v = (double*)xmalloc(sizeof(double) * (size_t)nnz);
  return a;
}
static void csr_free(csr* a) {
  if (!a) return;
  free(a->rp);
  free(a->ci);
  free(a->v);
  free(a);
}
static int64_t nnz_of(const csr* a) { return a->rp[a->n]; }

/* Growable builder (the push_back pattern used all over sparse.cpp). */
typedef struct {
  int64_t n, m, cap, len;
  int64_t* rp;
  int64_t* ci;
  double* v;
  int64_t row;
} builder;
static void b_init(builder* b, int64_t n, int64_t m, int64_t cap) {
  b->n = n;
  b->m = m;
  b->cap = cap > 16 ? cap : 16;
  b->len = 0;
  b->row = 0;
  b->rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
  b->ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)b->cap);
  b->v = (double*)xmalloc(sizeof(double) * (size_t)b->cap);
}
static void b_push(builder* b, int64_t c, double v) {
  if (b->len == b->cap) {
    b->cap *= 2;
    b->ci = (int64_t*)realloc(b->ci, sizeof(int64_t) * (size_t)b->cap);
    b->v = (double*)realloc(b->v, sizeof(double) * (size_t)b->cap);
    if (!b->ci || !b->v) fail(4, "out of memory");
  }
  b->ci[b->len] = c;
  b->v[b->len] = v;
  b->len++;
}
static void b_close_row(builder* b) { b->rp[++b->row] = b->len; }
static csr* b_finish(builder* b) {
  csr* a = (csr*)xcalloc(1, sizeof(csr));
  a->n = b->n;
  a->m = b->m;
  a->rp = b->rp;
  a->ci = b->ci;
  a->v = b->v;
  return a;
}

/* ctor validation, sparse.cpp:27-45 */
static void csr_validate(const csr* a) {
  if (a->n < 0 || a->m < 0) EINV("SparseMatrix: negative dimension");
  if (a->rp[0] != 0) EINV("SparseMatrix: row_offsets[0] must be 0");
  for (int64_t i = 0; i < a->n; ++i) {
    if (a->rp[i] > a->rp[i + 1]) EINV("SparseMatrix: row_offsets not monotone");
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      if (a->ci[k] < 0 || a->ci[k] >= a->m) EINV("SparseMatrix: column index out of range");
      if (k > a->rp[i] && !(a->ci[k - 1] < a->ci[k]))
        EINV("SparseMatrix: column indices not strictly increasing within row");
    }
  }
  for (int64_t k = 0; k < nnz_of(a); ++k)
    if (isnan(a->v[k])) EINV("SparseMatrix: stored NaN value");
}

static csr* csr_copy(const csr* a) {
  csr* b = csr_new(a->n, a->m, nnz_of(a));
  memcpy(b->rp, a->rp, sizeof(int64_t) * (size_t)(a->n + 1));
  memcpy(b->ci, a->ci, sizeof(int64_t) * (size_t)nnz_of(a));
  memcpy(b->v, a->v, sizeof(double) * (size_t)nnz_of(a));
  return b;
}

/* with_full_diagonal, sparse.cpp:132-160 */
static csr* with_full_diagonal(const csr* a) {
  if (a->n != a->m) EINV("SparseMatrix: with_full_diagonal requires a square matrix");
  builder b;
  b_init(&b, a->n, a->m, nnz_of(a) + a->n);
  for (int64_t i = 0; i < a->n; ++i) {
    int seen = 0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      const int64_t c = a->ci[k];
      if (!seen && c > i) {
        b_push(&b, i, 0.0);
        seen = 1;
      }
      if (c == i) seen = 1;
      b_push(&b, c, a->v[k]);
    }
    if (!seen) b_push(&b, i, 0.0);
    b_close_row(&b);
  }
  return b_finish(&b);
}

/* spmv, sparse.cpp:185-201 */
static void spmv_into(const csr* a, const double* x, double* y) {
  for (int64_t i = 0; i < a->n; ++i) {
    double acc = 0.0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) acc += a->v[k] * x[a->ci[k]];
    y[i] = acc;
  }
}

static int cmp_i64(const void* x, const void* y) {
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

/* spgemm, sparse.cpp:203-242 (Gustavson, dense work/stamp, sorted pattern) */
static csr* spgemm(const csr* a, const csr* b) {
  if (a->m != b->n) EINV("spgemm: dimension mismatch");
  const int64_t n = a->n, m = b->m;
  builder out;
  b_init(&out, n, m, nnz_of(a) * 2);
  double* work = (double*)xcalloc((size_t)m, sizeof(double));
  int64_t* stamp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(m ? m : 1));
  for (int64_t c = 0; c < m; ++c) stamp[c] = -1;
  int64_t cap = 64, len = 0;
  int64_t* pat = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)cap);
  for (int64_t i = 0; i < n; ++i) {
    len = 0;
    for (int64_t ak = a->rp[i]; ak < a->rp[i + 1]; ++ak) {
      const double av = a->v[ak];
      const int64_t j = a->ci[ak];
      for (int64_t bk = b->rp[j]; bk < b->rp[j + 1]; ++bk) {
        const int64_t c = b->ci[bk];
        if (stamp[c] != i) {
          stamp[c] = i;
          work[c] = 0.0;
          if (len == cap) {
            cap *= 2;
            pat = (int64_t*)realloc(pat, sizeof(int64_t) * (size_t)cap);
          }
          pat[len++] = c;
        }
        work[c] += av * b->v[bk];
      }
    }
    qsort(pat, (size_t)len, sizeof(int64_t), cmp_i64);
    for (int64_t k = 0; k < len; ++k) b_push(&out, pat[k], work[pat[k]]);
    b_close_row(&out);
  }
  free(work);
  free(stamp);
  free(pat);
  return b_finish(&out);
}

/* drop_entries, sparse.cpp:244-268 */
static csr* drop_entries(const csr* a, double tol, int keep_diagonal) {
  if (tol < 0.0) EINV("drop_entries: tol must be >= 0");
  const int square = keep_diagonal && a->n == a->m;
  builder b;
  b_init(&b, a->n, a->m, nnz_of(a));
  for (int64_t i = 0; i < a->n; ++i) {
    double row_max = 0.0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) row_max = fmax(row_max, fabs(a->v[k]));
    const double threshold = tol * row_max;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      const double mag = fabs(a->v[k]);
      const int diag = square && a->ci[k] == i;
      if (!diag && mag < threshold && mag < row_max) continue;
      b_push(&b, a->ci[k], a->v[k]);
    }
    b_close_row(&b);
  }
  return b_finish(&b);
}

/* ------------------------------------------------------------------------ */
/* LabelMap / extract_blocks, sparse.cpp:270-340 */
typedef struct {
  int64_t n, nf, nc;
  uint8_t* label;
  int64_t* fine_to_sub;
  int64_t* f_to_fine;
  int64_t* c_to_fine;
} labelmap;

static void map_free(labelmap* m) {
  free(m->label);
  free(m->fine_to_sub);
  free(m->f_to_fine);
  free(m->c_to_fine);
  memset(m, 0, sizeof *m);
}

static labelmap build_label_map(const uint8_t* labels, int64_t n) {
  labelmap m;
  m.n = n;
  m.nf = m.nc = 0;
  m.label = (uint8_t*)xmalloc((size_t)n);
  memcpy(m.label, labels, (size_t)n);
  m.fine_to_sub = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
  m.f_to_fine = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
  m.c_to_fine = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    if (labels[i] == AIRG_F) {
      m.fine_to_sub[i] = m.nf;
      m.f_to_fine[m.nf++] = i;
    } else if (labels[i] == AIRG_C) {
      m.fine_to_sub[i] = m.nc;
      m.c_to_fine[m.nc++] = i;
    } else {
      EINV("build_label_map: unassigned label at row %lld", (long long)i);
    }
  }
  return m;
}

typedef struct {
  csr *ff, *fc, *cf, *cc;
  labelmap map;
} blocksplit;

static void split_free(blocksplit* s) {
  csr_free(s->ff);
  csr_free(s->fc);
  csr_free(s->cf);
  csr_free(s->cc);
  map_free(&s->map);
}

static blocksplit extract_blocks(const csr* a, const uint8_t* labels) {
  blocksplit s;
  if (a->n != a->m) EINV("extract_blocks: label length mismatch");
  s.map = build_label_map(labels, a->n);
  const labelmap* map = &s.map;
  builder ff, fc, cf, cc;
  const int64_t nf = map->nf, nc = map->nc;
  b_init(&ff, nf, nf, 16);
  b_init(&fc, nf, nc, 16);
  b_init(&cf, nc, nf, 16);
  b_init(&cc, nc, nc, 16);
  for (int64_t i = 0; i < a->n; ++i) {
    const int row_f = map->label[i] == AIRG_F;
    builder* left = row_f ? &ff : &cf;
    builder* right = row_f ? &fc : &cc;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      const int64_t j = a->ci[k];
      if (map->label[j] == AIRG_F)
        b_push(left, map->fine_to_sub[j], a->v[k]);
      else
        b_push(right, map->fine_to_sub[j], a->v[k]);
    }
    b_close_row(left);
    b_close_row(right);
  }
  s.ff = b_finish(&ff);
  s.fc = b_finish(&fc);
  s.cf = b_finish(&cf);
  s.cc = b_finish(&cc);
  return s;
}

/* ------------------------------------------------------------------------ */
/* StrengthGraph, coarsening.hpp:14-41; strength coarsening.cpp:83-105;
 * finish_graph coarsening.cpp:28-42 (S rows come out sorted and unique
 * because A's columns are; S^T rows are filled in ascending i). */
typedef struct {
  int64_t n;
  int64_t *s_rp, *s_ci, *st_rp, *st_ci, *sym_rp, *sym_ci;
} sgraph;

static void graph_free(sgraph* g) {
  free(g->s_rp);
  free(g->s_ci);
  free(g->st_rp);
  free(g->st_ci);
  free(g->sym_rp);
  free(g->sym_ci);
}

static void finish_graph(sgraph* g) {
  const int64_t n = g->n, ns = g->s_rp[n];
  g->st_rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t k = 0; k < ns; ++k) g->st_rp[g->s_ci[k] + 1]++;
  for (int64_t j = 0; j < n; ++j) g->st_rp[j + 1] += g->st_rp[j];
  g->st_ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(ns ? ns : 1));
  int64_t* cur = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t j = 0; j < n; ++j) cur[j] = g->st_rp[j];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = g->s_rp[i]; k < g->s_rp[i + 1]; ++k) g->st_ci[cur[g->s_ci[k]]++] = i;
  free(cur);
  /* sym = sorted union of the two sorted rows */
  g->sym_rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
  g->sym_ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(2 * ns + 1));
  int64_t len = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = g->s_rp[i], ae = g->s_rp[i + 1], b = g->st_rp[i], be = g->st_rp[i + 1];
    while (a < ae || b < be) {
      int64_t v;
      if (b >= be || (a < ae && g->s_ci[a] < g->st_ci[b]))
        v = g->s_ci[a++];
      else if (a >= ae || g->st_ci[b] < g->s_ci[a])
        v = g->st_ci[b++];
      else {
        v = g->s_ci[a++];
        b++;
      }
      g->sym_ci[len++] = v;
    }
    g->sym_rp[i + 1] = len;
  }
}

static sgraph strength(const csr* a, double alpha) {
  if (a->n != a->m) EINV("strength: matrix must be square");
  sgraph g;
  memset(&g, 0, sizeof g);
  g.n = a->n;
  g.s_rp = (int64_t*)xcalloc((size_t)a->n + 1, sizeof(int64_t));
  g.s_ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(nnz_of(a) ? nnz_of(a) : 1));
  int64_t len = 0;
  for (int64_t i = 0; i < a->n; ++i) {
    double off_max = 0.0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k)
      if (a->ci[k] != i) off_max = fmax(off_max, fabs(a->v[k]));
    const double threshold = alpha * off_max;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      const double mag = fabs(a->v[k]);
      if (a->ci[k] != i && mag > 0.0 && mag >= threshold) g.s_ci[len++] = a->ci[k];
    }
    g.s_rp[i + 1] = len;
  }
  finish_graph(&g);
  return g;
}

/* weight_less coarsening.cpp:46-48; make_weights :50-63 */
static int weight_less(const double* w, int64_t i, int64_t j) {
  return w[i] != w[j] ? w[i] < w[j] : i < j;
}
static double* make_weights(const sgraph* g, uint64_t seed, int mode) {
  double* w = (double*)xmalloc(sizeof(double) * (size_t)(g->n ? g->n : 1));
  const uint64_t s = mix(seed, kStreamWeights);
  for (int64_t i = 0; i < g->n; ++i) {
    double deg;
    if (mode == 0)
      deg = (double)((g->s_rp[i + 1] - g->s_rp[i]) + (g->st_rp[i + 1] - g->st_rp[i]));
    else
      deg = (double)(g->sym_rp[i + 1] - g->sym_rp[i]);
    w[i] = deg + uniform01(s, (uint64_t)i);
  }
  return w;
}

/* pmisr_with_weights, coarsening.cpp:107-160 */
static void pmisr_with_weights(const sgraph* g, int64_t max_loops, const double* w,
                               uint8_t* label) {
  if (max_loops < 1) EINV("pmisr: max_loops must be >= 1");
  const int64_t n = g->n;
  int64_t unassigned = n;
  for (int64_t i = 0; i < n; ++i) {
    label[i] = AIRG_UNASSIGNED;
    if (w[i] < 1.0) {
      label[i] = AIRG_F;
      --unassigned;
    }
  }
  int64_t* d = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t loop = 0; loop < max_loops && unassigned > 0; ++loop) {
    int64_t nd = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (label[i] != AIRG_UNASSIGNED) continue;
      int minimal = 1;
      for (int64_t k = g->sym_rp[i]; k < g->sym_rp[i + 1]; ++k)
        if (!weight_less(w, i, g->sym_ci[k])) {
          minimal = 0;
          break;
        }
      if (minimal) d[nd++] = i;
    }
    if (nd == 0) break;
    for (int64_t t = 0; t < nd; ++t) {
      label[d[t]] = AIRG_F;
      --unassigned;
    }
    for (int64_t t = 0; t < nd; ++t)
      for (int64_t k = g->sym_rp[d[t]]; k < g->sym_rp[d[t] + 1]; ++k) {
        const int64_t j = g->sym_ci[k];
        if (label[j] == AIRG_UNASSIGNED) {
          label[j] = AIRG_C;
          --unassigned;
        }
      }
  }
  for (int64_t i = 0; i < n; ++i)
    if (label[i] == AIRG_UNASSIGNED) label[i] = AIRG_C;
  free(d);
}

/* ------------------------------------------------------------------------ */
/* dominance_report, coarsening.cpp:219-250 */
typedef struct {
  double* theta;
  double max_theta, alpha_diag;
  int64_t* hist;
  int64_t bins, n;
} domrep;

static domrep dominance_report(const csr* aff, int64_t bins) {
  if (bins < 1) EINV("dominance_report: bins >= 1");
  domrep r;
  r.n = aff->n;
  r.bins = bins;
  r.max_theta = 0.0;
  r.alpha_diag = 0.0;
  r.theta = (double*)xmalloc(sizeof(double) * (size_t)(aff->n ? aff->n : 1));
  for (int64_t i = 0; i < aff->n; ++i) {
    double off = 0.0, diag = 0.0;
    int seen = 0;
    for (int64_t k = aff->rp[i]; k < aff->rp[i + 1]; ++k) {
      if (aff->ci[k] == i) {
        diag = fabs(aff->v[k]);
        seen = 1;
      } else {
        off += fabs(aff->v[k]);
      }
    }
    if (!seen || diag == 0.0) {
      free(r.theta);
      ERUN("dominance_report: zero diagonal in A_ff row %lld", (long long)i);
    }
    r.theta[i] = off / diag;
    r.max_theta = fmax(r.max_theta, r.theta[i]);
  }
  r.hist = (int64_t*)xcalloc((size_t)bins, sizeof(int64_t));
  const double width = r.max_theta > 0.0 ? r.max_theta / (double)bins : 1.0;
  for (int64_t i = 0; i < aff->n; ++i) {
    int64_t b = (int64_t)(r.theta[i] / width);
    ++r.hist[b < bins - 1 ? b : bins - 1];
  }
  return r;
}
static void domrep_free(domrep* r) {
  free(r->theta);
  free(r->hist);
}

static int cmp_f64(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* ddc, coarsening.cpp:252-330. Converts in `label` (global rows); returns
 * the number converted. */
static int64_t ddc(const csr* aff, uint8_t* label, const labelmap* map, double fraction,
                   int64_t bins, int selection, double direct_alpha, domrep* rep_out) {
  if (aff->n != map->nf) EINV("ddc: a_ff does not match label map");
  if (fraction <= 0.0 || fraction > 1.0) EINV("ddc: fraction must be in (0, 1]");
  domrep rep = dominance_report(aff, bins);
  const int64_t nf = aff->n;
  double alpha_diag = 0.0;
  if (selection == 2) {
    alpha_diag = direct_alpha;
  } else if (selection == 1) {
    int64_t target = llround(fraction * (double)nf);
    if (target < 0) target = 0;
    if (target > nf) target = nf;
    if (target == 0 || rep.max_theta == 0.0) {
      alpha_diag = rep.max_theta;
    } else if (target == nf) {
      alpha_diag = -1.0;
    } else {
      double* s = (double*)xmalloc(sizeof(double) * (size_t)nf);
      memcpy(s, rep.theta, sizeof(double) * (size_t)nf);
      qsort(s, (size_t)nf, sizeof(double), cmp_f64);
      alpha_diag = s[(nf - target) - 1];
      free(s);
    }
  } else {
    const double max_theta = rep.max_theta;
    if (max_theta == 0.0) {
      alpha_diag = 0.0;
    } else {
      const double target = fraction * (double)nf;
      int64_t above = 0, best_k = bins;
      double best_err = fabs((double)above - target);
      for (int64_t k = bins; k-- > 0;) {
        above += rep.hist[k];
        const double err = fabs((double)above - target);
        if (err < best_err) {
          best_err = err;
          best_k = k;
        }
      }
      alpha_diag = (double)best_k * (max_theta / (double)bins);
    }
  }
  rep.alpha_diag = alpha_diag;
  int64_t converted = 0;
  for (int64_t k = 0; k < nf; ++k)
    if (rep.theta[k] > alpha_diag && rep.theta[k] != 0.0) {
      label[map->f_to_fine[k]] = AIRG_C;
      ++converted;
    }
  if (rep_out)
    *rep_out = rep;
  else
    domrep_free(&rep);
  return converted;
}

/* ------------------------------------------------------------------------ */
/* power_pattern, gmres_poly.cpp:18-59: pattern(A^s) u I u pattern(A). */
static csr* power_pattern(const csr* a, int64_t s) {
  const int64_t n = a->n;
  csr* cur = csr_copy(a);
  int64_t* stamp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t k = 1; k < s; ++k) {
    for (int64_t i = 0; i < n; ++i) stamp[i] = -1;
    builder nb;
    b_init(&nb, n, n, nnz_of(cur) * 2);
    int64_t cap = 64, len;
    int64_t* scr = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)cap);
    for (int64_t i = 0; i < n; ++i) {
      len = 0;
      for (int64_t t = cur->rp[i]; t < cur->rp[i + 1]; ++t) {
        const int64_t j = cur->ci[t];
        for (int64_t q = a->rp[j]; q < a->rp[j + 1]; ++q) {
          const int64_t c = a->ci[q];
          if (stamp[c] != i) {
            stamp[c] = i;
            if (len == cap) {
              cap *= 2;
              scr = (int64_t*)realloc(scr, sizeof(int64_t) * (size_t)cap);
            }
            scr[len++] = c;
          }
        }
      }
      qsort(scr, (size_t)len, sizeof(int64_t), cmp_i64);
      for (int64_t t = 0; t < len; ++t) b_push(&nb, scr[t], 0.0);
      b_close_row(&nb);
    }
    free(scr);
    csr_free(cur);
    cur = b_finish(&nb);
  }
  free(stamp);
  /* insert the diagonal, then union with pattern(A) */
  builder out;
  b_init(&out, n, n, nnz_of(cur) + n + nnz_of(a));
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = cur->rp[i], pe = cur->rp[i + 1], q = a->rp[i], qe = a->rp[i + 1];
    int diag_done = 0;
    int64_t last = -1;
    while (p < pe || q < qe || !diag_done) {
      int64_t cand = INT64_MAX;
      if (p < pe) cand = cur->ci[p];
      if (q < qe && a->ci[q] < cand) cand = a->ci[q];
      if (!diag_done && i < cand) cand = i;
      if (cand == i) diag_done = 1;
      if (p < pe && cur->ci[p] == cand) ++p;
      if (q < qe && a->ci[q] == cand) ++q;
      if (cand != last) b_push(&out, cand, 0.0);
      last = cand;
    }
    b_close_row(&out);
  }
  csr_free(cur);
  return b_finish(&out);
}

/* assemble_fixed_sparsity, gmres_poly.cpp:197-280 */
static csr* assemble_fixed_sparsity(const csr* a, const double* coeffs, int64_t ncoeffs,
                                    int64_t deg, int64_t sparsity_order, uint64_t* flops_out) {
  if (a->n != a->m) EINV("assemble_fixed_sparsity: square matrix only");
  if (sparsity_order < 1) EINV("assemble_fixed_sparsity: sparsity_order >= 1");
  if (ncoeffs < 1) EINV("assemble_fixed_sparsity: empty polynomial");
  const int64_t n = a->n;
  csr* pat = power_pattern(a, sparsity_order);
  csr* out = pat; /* reuse pattern arrays for the output */
  int64_t* pos = (int64_t*)xcalloc((size_t)(n ? n : 1), sizeof(int64_t));
  int64_t* stamp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) stamp[i] = -1;
  int64_t wmax = 1;
  for (int64_t i = 0; i < n; ++i)
    if (pat->rp[i + 1] - pat->rp[i] > wmax) wmax = pat->rp[i + 1] - pat->rp[i];
  double* cur = (double*)xmalloc(sizeof(double) * (size_t)wmax);
  double* next = (double*)xmalloc(sizeof(double) * (size_t)wmax);
  uint64_t flops = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t o = pat->rp[i], width = pat->rp[i + 1] - o;
    for (int64_t k = 0; k < width; ++k) {
      pos[pat->ci[o + k]] = k;
      stamp[pat->ci[o + k]] = i;
    }
    double* ov = out->v + o;
    for (int64_t k = 0; k < width; ++k) ov[k] = (pat->ci[o + k] == i) ? coeffs[0] : 0.0;
    for (int64_t k = 0; k < width; ++k) cur[k] = 0.0;
    for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
      cur[pos[a->ci[k]]] = a->v[k];
      if (deg >= 1) {
        ov[pos[a->ci[k]]] += coeffs[1] * a->v[k];
        flops += 2;
      }
    }
    for (int64_t power = 2; power <= deg; ++power) {
      for (int64_t k = 0; k < width; ++k) next[k] = 0.0;
      for (int64_t k = 0; k < width; ++k) {
        const double v = cur[k];
        if (v == 0.0) continue;
        const int64_t j = pat->ci[o + k];
        for (int64_t t = a->rp[j]; t < a->rp[j + 1]; ++t) {
          const int64_t c = a->ci[t];
          if (stamp[c] != i) continue;
          next[pos[c]] += v * a->v[t];
          flops += 2;
        }
      }
      const double alpha = coeffs[power];
      for (int64_t k = 0; k < width; ++k) {
        ov[k] += alpha * next[k];
        flops += 2;
      }
      double* t = cur;
      cur = next;
      next = t;
    }
  }
  free(pos);
  free(stamp);
  free(cur);
  free(next);
  if (flops_out) *flops_out += flops;
  return out;
}

/* ------------------------------------------------------------------------ */
/* compute_coefficients, gmres_poly.cpp:63-171, in long double. Dense
 * matrices are column-major. The QR / COD follow oracle/shim/Eigen/Dense
 * operation for operation. */
typedef long double ld;

static void make_householder(const ld* x, int64_t n, ld* v, ld* tau, ld* beta) {
  for (int64_t i = 0; i < n; ++i) v[i] = x[i];
  ld tail = 0;
  for (int64_t i = 1; i < n; ++i) tail += x[i] * x[i];
  const ld c0 = x[0];
  if (tail <= LDBL_MIN) {
    *tau = 0;
    *beta = c0;
    for (int64_t i = 1; i < n; ++i) v[i] = 0;
    v[0] = 1;
    return;
  }
  ld b = sqrtl(c0 * c0 + tail);
  if (c0 >= 0) b = -b;
  for (int64_t i = 1; i < n; ++i) v[i] = x[i] / (c0 - b);
  v[0] = 1;
  *tau = (b - c0) / b;
  *beta = b;
}

/* rows [r0, r0+nv) of columns [c0, c1) of an (lda x *) column-major matrix */
static void apply_left(ld* a, int64_t lda, int64_t r0, const ld* v, int64_t nv, ld tau,
                       int64_t c0, int64_t c1) {
  if (tau == 0) return;
  for (int64_t j = c0; j < c1; ++j) {
    ld s = 0;
    for (int64_t i = 0; i < nv; ++i) s += v[i] * a[(r0 + i) + j * lda];
    s *= tau;
    for (int64_t i = 0; i < nv; ++i) a[(r0 + i) + j * lda] -= s * v[i];
  }
}

/* Minimum-norm least squares min ||A x - b|| through column-pivoted QR + RZ
 * (shim CompleteOrthogonalDecomposition). Returns the rank; x gets n. */
static int64_t cod_solve(const ld* A, int64_t m, int64_t n, ld thr, const ld* b, ld* x) {
  ld* t = (ld*)xmalloc(sizeof(ld) * (size_t)(m * n + 1));
  memcpy(t, A, sizeof(ld) * (size_t)(m * n));
  int64_t* perm = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < n; ++j) perm[j] = j;
  const int64_t k = m < n ? m : n;
  const int64_t vmax = (m > n ? m : n) + 2;
  ld* hv = (ld*)xmalloc(sizeof(ld) * (size_t)(k * vmax + 1));
  int64_t* hn = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(k + 1));
  ld* htau = (ld*)xmalloc(sizeof(ld) * (size_t)(k + 1));
  ld* xs = (ld*)xmalloc(sizeof(ld) * (size_t)vmax);
  ld maxpivot = 0;
#define T_(i, j) t[(i) + (j) * m]
  for (int64_t j = 0; j < k; ++j) {
    int64_t best = j;
    ld bestn = -1;
    for (int64_t c = j; c < n; ++c) {
      ld s = 0;
      for (int64_t i = j; i < m; ++i) s += T_(i, c) * T_(i, c);
      if (s > bestn) {
        bestn = s;
        best = c;
      }
    }
    if (best != j) {
      for (int64_t i = 0; i < m; ++i) {
        ld tmp = T_(i, j);
        T_(i, j) = T_(i, best);
        T_(i, best) = tmp;
      }
      int64_t tp = perm[j];
      perm[j] = perm[best];
      perm[best] = tp;
    }
    for (int64_t i = j; i < m; ++i) xs[i - j] = T_(i, j);
    ld tau, beta;
    make_householder(xs, m - j, hv + j * vmax, &tau, &beta);
    hn[j] = m - j;
    htau[j] = tau;
    apply_left(t, m, j, hv + j * vmax, m - j, tau, j + 1, n);
    T_(j, j) = beta;
    for (int64_t i = j + 1; i < m; ++i) T_(i, j) = 0;
    if (fabsl(beta) > maxpivot) maxpivot = fabsl(beta);
  }
  int64_t rank = 0;
  for (int64_t j = 0; j < k; ++j)
    if (fabsl(T_(j, j)) > thr * maxpivot) ++rank;
  /* RZ on the top rank rows */
  const int64_t zl = 1 + (n - rank);
  ld* zv = (ld*)xmalloc(sizeof(ld) * (size_t)((rank + 1) * (zl + 1)));
  ld* ztau = (ld*)xcalloc((size_t)(rank + 1), sizeof(ld));
  if (rank < n) {
    for (int64_t kk = rank - 1; kk >= 0; --kk) {
      xs[0] = T_(kk, kk);
      for (int64_t c = rank; c < n; ++c) xs[1 + c - rank] = T_(kk, c);
      ld tau, beta;
      ld* v = zv + kk * (zl + 1);
      make_householder(xs, zl, v, &tau, &beta);
      for (int64_t r = 0; r <= kk; ++r) {
        ld s = T_(r, kk) * v[0];
        for (int64_t c = rank; c < n; ++c) s += T_(r, c) * v[1 + c - rank];
        s *= tau;
        T_(r, kk) -= s * v[0];
        for (int64_t c = rank; c < n; ++c) T_(r, c) -= s * v[1 + c - rank];
      }
      ztau[kk] = tau;
    }
  }
  /* solve */
  ld* c = (ld*)xmalloc(sizeof(ld) * (size_t)(m + 1));
  for (int64_t i = 0; i < m; ++i) c[i] = b[i];
  for (int64_t j = 0; j < k; ++j) {
    const ld* v = hv + j * vmax;
    ld s = 0;
    for (int64_t i = 0; i < hn[j]; ++i) s += v[i] * c[j + i];
    s *= htau[j];
    for (int64_t i = 0; i < hn[j]; ++i) c[j + i] -= s * v[i];
  }
  ld* w = (ld*)xcalloc((size_t)(n + 1), sizeof(ld));
  for (int64_t i = rank - 1; i >= 0; --i) {
    ld s = c[i];
    for (int64_t j = i + 1; j < rank; ++j) s -= T_(i, j) * w[j];
    w[i] = s / T_(i, i);
  }
  for (int64_t i = rank; i < n; ++i) w[i] = 0;
  if (rank < n) {
    for (int64_t kk = 0; kk < rank; ++kk) {
      if (ztau[kk] == 0) continue;
      const ld* v = zv + kk * (zl + 1);
      ld s = w[kk] * v[0];
      for (int64_t i = 1; i < zl; ++i) s += v[i] * w[rank + i - 1];
      s *= ztau[kk];
      w[kk] -= s * v[0];
      for (int64_t i = 1; i < zl; ++i) w[rank + i - 1] -= s * v[i];
    }
  }
  for (int64_t j = 0; j < n; ++j) x[perm[j]] = w[j];
#undef T_
  free(t);
  free(perm);
  free(hv);
  free(hn);
  free(htau);
  free(xs);
  free(zv);
  free(ztau);
  free(c);
  free(w);
  return rank;
}

static void compute_coefficients(const csr* a, int64_t m, uint64_t seed, double* coeffs,
                                 int64_t* eff_order) {
  if (a->n != a->m) EINV("compute_coefficients: matrix must be square");
  if (m < 1) EINV("compute_coefficients: m must be >= 1");
  const int64_t n = a->n;
  if (n == 0) EINV("compute_coefficients: empty matrix");
  const int64_t nc = m + 1;
  const uint64_t rhs_seed = mix(seed, kStreamPolyRhs);
  ld* basis = (ld*)xmalloc(sizeof(ld) * (size_t)(n * nc));
#define B_(i, k) basis[(i) + (k) * n]
  for (int64_t i = 0; i < n; ++i) B_(i, 0) = (ld)standard_normal(rhs_seed, (uint64_t)i);
  for (int64_t k = 1; k <= m; ++k)
    for (int64_t i = 0; i < n; ++i) {
      ld acc = 0;
      for (int64_t t = a->rp[i]; t < a->rp[i + 1]; ++t) acc += (ld)a->v[t] * B_(a->ci[t], k - 1);
      B_(i, k) = acc;
    }
  ld* scale = (ld*)xmalloc(sizeof(ld) * (size_t)nc);
  for (int64_t k = 0; k <= m; ++k) {
    ld s = 0;
    for (int64_t i = 0; i < n; ++i) s += B_(i, k) * B_(i, k);
    scale[k] = sqrtl(s);
    if (scale[k] > 0)
      for (int64_t i = 0; i < n; ++i) B_(i, k) /= scale[k];
  }
  if (scale[0] == 0) ERUN("compute_coefficients: zero right-hand side");
  const int64_t rrows = n < nc ? n : nc;
  /* Householder QR of a copy of the normalised basis */
  ld* qr = (ld*)xmalloc(sizeof(ld) * (size_t)(n * nc));
  memcpy(qr, basis, sizeof(ld) * (size_t)(n * nc));
  {
    const int64_t kk = n < nc ? n : nc;
    ld* v = (ld*)xmalloc(sizeof(ld) * (size_t)(n + 1));
    ld* x = (ld*)xmalloc(sizeof(ld) * (size_t)(n + 1));
    for (int64_t j = 0; j < kk; ++j) {
      for (int64_t i = j; i < n; ++i) x[i - j] = qr[i + j * n];
      ld tau, beta;
      make_householder(x, n - j, v, &tau, &beta);
      apply_left(qr, n, j, v, n - j, tau, j + 1, nc);
      qr[j + j * n] = beta;
    }
    free(v);
    free(x);
  }
  /* r_scaled = upper triangle of the top rrows rows */
  ld* r = (ld*)xcalloc((size_t)(rrows * nc), sizeof(ld));
#define R_(i, k) r[(i) + (k) * rrows]
  for (int64_t k = 0; k < nc; ++k)
    for (int64_t i = 0; i < rrows && i <= k; ++i) R_(i, k) = qr[i + k * n];
  free(qr);
  int64_t dim = 0;
  for (int64_t k = 0; k < rrows; ++k) {
    if (fabs((double)R_(k, k)) < 1e-12) break;
    ++dim;
  }
  if (dim == 0) ERUN("compute_coefficients: singular projected system");
  for (int64_t k = 0; k <= m; ++k)
    for (int64_t i = 0; i < rrows; ++i) R_(i, k) *= scale[k];
  const int64_t lcols = m < dim ? m : dim;
  ld* b0 = (ld*)xmalloc(sizeof(ld) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) b0[i] = B_(i, 0) * scale[0];
  ld* aqb = (ld*)xmalloc(sizeof(ld) * (size_t)n);
  ld* y = (ld*)xmalloc(sizeof(ld) * (size_t)(m + 1));
  ld* best_y = (ld*)xcalloc((size_t)(m + 1), sizeof(ld));
  ld* rt = (ld*)xmalloc(sizeof(ld) * (size_t)((rrows + 1) * (m + 1)));
  ld* rhs = (ld*)xmalloc(sizeof(ld) * (size_t)(rrows + 2));
  int64_t best_d = 0;
  ld best_resid = (ld)INFINITY;
  for (int64_t d = 1; d <= lcols; ++d) {
    const int64_t lrows = rrows < d + 1 ? rrows : d + 1;
    for (int64_t j = 0; j < d; ++j)
      for (int64_t i = 0; i < lrows; ++i) rt[i + j * lrows] = R_(i, 1 + j);
    for (int64_t i = 0; i < lrows; ++i) rhs[i] = 0;
    rhs[0] = R_(0, 0);
    const int64_t rank = cod_solve(rt, lrows, d, (ld)1e-12, rhs, y);
    if (rank == 0) continue;
    int finite = 1;
    for (int64_t k = 0; k < d; ++k)
      if (!isfinite(y[k])) finite = 0;
    if (!finite) continue;
    for (int64_t i = 0; i < n; ++i) aqb[i] = 0;
    for (int64_t k = 0; k < d; ++k) {
      const ld s = y[k] * scale[k + 1];
      for (int64_t i = 0; i < n; ++i) aqb[i] += B_(i, k + 1) * s;
    }
    ld ss = 0;
    for (int64_t i = 0; i < n; ++i) {
      const ld df = b0[i] - aqb[i];
      ss += df * df;
    }
    const ld resid = sqrtl(ss) / scale[0];
    if (resid < best_resid) {
      best_resid = resid;
      best_d = d;
      for (int64_t k = 0; k < d; ++k) best_y[k] = y[k];
    }
  }
  if (best_d == 0) ERUN("compute_coefficients: singular projected system");
  for (int64_t k = 0; k < m; ++k) coeffs[k] = 0.0;
  for (int64_t k = 0; k < best_d; ++k) coeffs[k] = (double)best_y[k];
  *eff_order = best_d - 1;
#undef B_
#undef R_
  free(basis);
  free(scale);
  free(r);
  free(b0);
  free(aqb);
  free(y);
  free(best_y);
  free(rt);
  free(rhs);
}

/* ------------------------------------------------------------------------ */
/* smoother_growth_estimate air.cpp:61-95; make_checked_inverse :106-129 */
static double smoother_growth_estimate(const csr* a, const csr* q) {
  const int64_t n = a->n;
  if (n == 0) return 0.0;
  const uint64_t probe_seed = mix(0xA3B1C5D7ull, (uint64_t)n);
  double* v = (double*)xmalloc(sizeof(double) * (size_t)n);
  double* av = (double*)xmalloc(sizeof(double) * (size_t)n);
  double* qav = (double*)xmalloc(sizeof(double) * (size_t)n);
  double norm = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    v[i] = standard_normal(probe_seed, (uint64_t)i);
    norm += v[i] * v[i];
  }
  norm = sqrt(norm);
  for (int64_t i = 0; i < n; ++i) v[i] /= norm;
  double log_growth = 0.0;
  int tail = 0;
  double result = -1.0;
  for (int k = 0; k < 30; ++k) {
    spmv_into(a, v, av);
    spmv_into(q, av, qav);
    double g = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      v[i] -= qav[i];
      g += v[i] * v[i];
    }
    g = sqrt(g);
    if (g == 0.0) {
      result = 0.0;
      break;
    }
    for (int64_t i = 0; i < n; ++i) v[i] /= g;
    if (k >= 15) {
      log_growth += log(g);
      ++tail;
    }
  }
  if (result < 0.0) result = exp(log_growth / tail);
  free(v);
  free(av);
  free(qav);
  return result;
}

typedef struct {
  double coeffs[32];
  int64_t ncoeffs, eff;
  csr* assembled;
  double growth;
  int64_t attempts;
} checked_inv;

static checked_inv make_checked_inverse(const csr* a, int64_t order, int64_t sparsity,
                                        uint64_t seed) {
  checked_inv best;
  memset(&best, 0, sizeof best);
  double best_growth = INFINITY;
  for (int64_t attempt = 0; attempt < 6; ++attempt) {
    const uint64_t s = attempt == 0 ? seed : mix(seed, 0x52455452ull + (uint64_t)attempt);
    double c[32];
    int64_t eff;
    compute_coefficients(a, order + 1, s, c, &eff);
    csr* q = assemble_fixed_sparsity(a, c, order + 1, eff, sparsity, NULL);
    const double growth = smoother_growth_estimate(a, q);
    if (growth < best_growth) {
      csr_free(best.assembled);
      memcpy(best.coeffs, c, sizeof(double) * (size_t)(order + 1));
      best.ncoeffs = order + 1;
      best.eff = eff;
      best.assembled = q;
      best.growth = growth;
      best.attempts = attempt + 1;
      best_growth = growth;
    } else {
      csr_free(q);
    }
    if (best_growth <= 0.5) break;
  }
  return best;
}

/* ------------------------------------------------------------------------ */
/* build_restriction air.cpp:154-189 */
typedef struct {
  int64_t col;
  double val;
} pair_cv;
static int cmp_pair(const void* x, const void* y) {
  const pair_cv* a = (const pair_cv*)x;
  const pair_cv* b = (const pair_cv*)y;
  if (a->col != b->col) return (a->col > b->col) - (a->col < b->col);
  return (a->val > b->val) - (a->val < b->val);
}
static csr* build_restriction(const csr* acf, const csr* ffinv, double drop, const labelmap* map) {
  csr* z0 = spgemm(acf, ffinv);
  csr* z = drop_entries(z0, drop, 0);
  csr_free(z0);
  builder b;
  b_init(&b, map->nc, map->n, nnz_of(z) + map->nc);
  pair_cv* row = (pair_cv*)xmalloc(sizeof(pair_cv) * (size_t)(z->m + 2));
  for (int64_t c = 0; c < map->nc; ++c) {
    int64_t len = 0;
    for (int64_t k = z->rp[c]; k < z->rp[c + 1]; ++k) {
      row[len].col = map->f_to_fine[z->ci[k]];
      row[len].val = -z->v[k];
      ++len;
    }
    row[len].col = map->c_to_fine[c];
    row[len].val = 1.0;
    ++len;
    qsort(row, (size_t)len, sizeof(pair_cv), cmp_pair);
    for (int64_t k = 0; k < len; ++k) b_push(&b, row[k].col, row[k].val);
    b_close_row(&b);
  }
  free(row);
  csr_free(z);
  return b_finish(&b);
}

/* entry lookup, sparse.cpp:102-107 */
static double csr_entry(const csr* a, int64_t i, int64_t j) {
  int64_t lo = a->rp[i], hi = a->rp[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (a->ci[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == a->rp[i + 1] || a->ci[lo] != j) return 0.0;
  return a->v[lo];
}

/* build_prolongation air.cpp:191-238 (one-point) */
static csr* build_prolongation(const uint8_t* label, const labelmap* map, const sgraph* g,
                               const csr* a) {
  const int64_t n = map->n;
  builder b;
  b_init(&b, n, map->nc, n);
  for (int64_t i = 0; i < n; ++i) {
    if (map->label[i] == AIRG_C) {
      b_push(&b, map->fine_to_sub[i], 1.0);
    } else {
      int64_t best = -1;
      double best_mag = -1.0;
      for (int64_t k = g->s_rp[i]; k < g->s_rp[i + 1]; ++k) {
        const int64_t j = g->s_ci[k];
        if (label[j] != AIRG_C) continue;
        const double mag = fabs(csr_entry(a, i, j));
        if (mag > best_mag) {
          best_mag = mag;
          best = j;
        }
      }
      if (best < 0) {
        for (int64_t k = a->rp[i]; k < a->rp[i + 1]; ++k) {
          const int64_t c = a->ci[k];
          if (c == i || label[c] != AIRG_C) continue;
          const double mag = fabs(a->v[k]);
          if (mag > best_mag) {
            best_mag = mag;
            best = c;
          }
        }
      }
      if (best >= 0) b_push(&b, map->fine_to_sub[best], 1.0);
    }
    b_close_row(&b);
  }
  return b_finish(&b);
}

/* coarse_matrix air.cpp:268-271 */
static csr* coarse_matrix(const csr* r, const csr* a, const csr* p, double drop) {
  csr* ap = spgemm(a, p);
  csr* rap = spgemm(r, ap);
  csr_free(ap);
  csr* out = drop_entries(rap, drop, 1);
  csr_free(rap);
  return out;
}

/* ------------------------------------------------------------------------ */
/* Hierarchy, air.hpp:49-91 */
typedef struct {
  csr *a, *aff, *afc, *acf, *ffinv, *r, *p;
  uint8_t* label;
  labelmap map;
  int64_t n_f_pre, n_converted;
  double max_theta_pre, alpha_diag, max_theta_post, growth;
  int64_t attempts, eff;
  double coeffs[32];
} level_t;

typedef struct {
  int64_t nlev, cap;
  level_t* lev;
  csr* coarse_a;
  csr* coarse_inv;
  double coarse_coeffs[32];
  int64_t coarse_eff, coarse_attempts;
  double coarse_growth;
  int64_t coarse_iterations;
  double grid_c, op_c, store_c;
} hier_t;

static void level_free(level_t* l) {
  csr_free(l->a);
  csr_free(l->aff);
  csr_free(l->afc);
  csr_free(l->acf);
  csr_free(l->ffinv);
  csr_free(l->r);
  csr_free(l->p);
  free(l->label);
  map_free(&l->map);
}

static void hier_destroy(hier_t* h) {
  if (!h) return;
  for (int64_t l = 0; l < h->nlev; ++l) level_free(&h->lev[l]);
  free(h->lev);
  csr_free(h->coarse_a);
  csr_free(h->coarse_inv);
  free(h);
}

/* recompute_metrics air.cpp:412-434 */
static void recompute_metrics(hier_t* h) {
  const csr* top = h->nlev ? h->lev[0].a : h->coarse_a;
  const double n0 = (double)top->n, nnz0 = (double)nnz_of(top);
  double grid = 0.0, op = 0.0, store = 0.0;
  for (int64_t l = 0; l < h->nlev; ++l) {
    const level_t* L = &h->lev[l];
    grid += (double)L->a->n;
    op += (double)nnz_of(L->a);
    store += (double)(nnz_of(L->ffinv) + nnz_of(L->aff) + nnz_of(L->afc) + nnz_of(L->r) +
                      nnz_of(L->p));
  }
  grid += (double)h->coarse_a->n;
  op += (double)nnz_of(h->coarse_a);
  store += (double)nnz_of(h->coarse_inv);
  if (h->coarse_iterations > 1) store += (double)nnz_of(h->coarse_a);
  h->grid_c = grid / n0;
  h->op_c = op / nnz0;
  h->store_c = store / nnz0;
}

/* setup air.cpp:285-410 (one-point prolongation, PMISR/PMIS, no test hooks) */
static void pmis_with_weights(const sgraph* g, int swap, const double* w, uint8_t* label);

static hier_t* setup(const csr* a0, const airg_setup_config* cfg) {
  if (a0->n != a0->m) EINV("setup: matrix must be square");
  if (cfg->poly_order < 1 || cfg->coarse_poly_order < 1)
    EINV("setup: polynomial orders must be >= 1");
  if (cfg->sparsity_order < 1) EINV("setup: sparsity_order must be >= 1");
  if (cfg->drop_coarse < 0.0 || cfg->drop_restrict < 0.0)
    EINV("setup: drop tolerances must be >= 0");
  if (cfg->strength_alpha < 0.0 || cfg->strength_alpha > 1.0)
    EINV("setup: strength_alpha must lie in [0, 1]");
  if (cfg->prolongation != 0) EINV("setup: only one-point prolongation is restated");
  if (cfg->poly_order + 1 > 32 || cfg->coarse_poly_order + 1 > 32)
    EINV("setup: polynomial order above 31 not supported");
  hier_t* h = (hier_t*)xcalloc(1, sizeof(hier_t));
  h->coarse_iterations = cfg->coarse_iterations;
  h->cap = 8;
  h->lev = (level_t*)xcalloc((size_t)h->cap, sizeof(level_t));
  int have_coarse = 0;
  checked_inv cc;
  memset(&cc, 0, sizeof cc);
  csr* current = with_full_diagonal(a0);
  for (;;) {
    const int64_t built = h->nlev;
    const int forced = current->n <= cfg->poly_order + 1 ||
                       (cfg->max_levels > 0 && built + 1 >= cfg->max_levels);
    if (forced || current->n <= cfg->coarse_size_target) {
      const uint64_t s = mix(cfg->seed, 0xC0A12534ull + (uint64_t)built);
      cc = make_checked_inverse(current, cfg->coarse_poly_order, cfg->sparsity_order, s);
      have_coarse = 1;
      if (forced || cc.growth <= 0.5) break;
      csr_free(cc.assembled);
      memset(&cc, 0, sizeof cc);
      have_coarse = 0;
    }
    if (h->nlev == h->cap) {
      h->cap *= 2;
      h->lev = (level_t*)realloc(h->lev, sizeof(level_t) * (size_t)h->cap);
    }
    level_t* L = &h->lev[h->nlev];
    memset(L, 0, sizeof *L);
    L->a = current;
    current = NULL;
    const int64_t n = L->a->n;
    const uint64_t level_seed = mix(cfg->seed, (uint64_t)h->nlev);
    sgraph g = strength(L->a, cfg->strength_alpha);
    L->label = (uint8_t*)xmalloc((size_t)(n ? n : 1));
    double* w = make_weights(&g, level_seed, cfg->cf == 0 ? cfg->weight_mode : 0);
    if (cfg->cf == 0)
      pmisr_with_weights(&g, cfg->max_loops, w, L->label);
    else
      pmis_with_weights(&g, cfg->cf == 2, w, L->label);
    free(w);
    blocksplit split = extract_blocks(L->a, L->label);
    L->n_f_pre = split.map.nf;
    if (cfg->ddc_enabled && split.map.nf > 0) {
      domrep rep;
      const int64_t conv = ddc(split.ff, L->label, &split.map, cfg->ddc_fraction, cfg->ddc_bins,
                               0, 0.0, &rep);
      L->max_theta_pre = rep.max_theta;
      L->alpha_diag = rep.alpha_diag;
      domrep_free(&rep);
      L->n_converted = conv;
      if (conv > 0) {
        split_free(&split);
        split = extract_blocks(L->a, L->label);
      }
    } else {
      domrep rep = dominance_report(split.ff, cfg->ddc_bins);
      L->max_theta_pre = rep.max_theta;
      domrep_free(&rep);
    }
    {
      domrep rep = dominance_report(split.ff, cfg->ddc_bins);
      L->max_theta_post = rep.max_theta;
      domrep_free(&rep);
    }
    L->map = split.map;
    L->aff = split.ff;
    L->afc = split.fc;
    L->acf = split.cf;
    csr_free(split.cc);
    const int64_t nc = L->map.nc;
    if (L->map.nf == 0)
      ERUN("setup: coarsening stall, no F points selected on level %lld", (long long)h->nlev);
    if (nc == 0) {
      current = L->a;
      L->a = NULL;
      level_free(L);
      graph_free(&g);
      break;
    }
    if ((double)nc > 0.99 * (double)n)
      ERUN("setup: coarsening stall, level %lld coarsened by less than 1%% (%lld -> %lld)",
           (long long)h->nlev, (long long)n, (long long)nc);
    checked_inv ci = make_checked_inverse(L->aff, cfg->poly_order, cfg->sparsity_order, level_seed);
    L->ffinv = ci.assembled;
    L->growth = ci.growth;
    L->attempts = ci.attempts;
    L->eff = ci.eff;
    memcpy(L->coeffs, ci.coeffs, sizeof(double) * (size_t)ci.ncoeffs);
    L->r = build_restriction(L->acf, L->ffinv, cfg->drop_restrict, &L->map);
    L->p = build_prolongation(L->label, &L->map, &g, L->a);
    graph_free(&g);
    csr* cm = coarse_matrix(L->r, L->a, L->p, cfg->drop_coarse);
    current = with_full_diagonal(cm);
    csr_free(cm);
    h->nlev++;
  }
  h->coarse_a = current;
  if (!have_coarse) {
    const uint64_t s = mix(cfg->seed, 0xC0A12534ull + (uint64_t)h->nlev);
    cc = make_checked_inverse(h->coarse_a, cfg->coarse_poly_order, cfg->sparsity_order, s);
  }
  h->coarse_inv = cc.assembled;
  memcpy(h->coarse_coeffs, cc.coeffs, sizeof(double) * (size_t)cc.ncoeffs);
  h->coarse_eff = cc.eff;
  h->coarse_attempts = cc.attempts;
  h->coarse_growth = cc.growth;
  recompute_metrics(h);
  return h;
}

/* pmis_with_weights coarsening.cpp:169-210 (comparison baseline) */
static void pmis_with_weights(const sgraph* g, int swap, const double* w, uint8_t* label) {
  const int64_t n = g->n;
  for (int64_t i = 0; i < n; ++i) label[i] = AIRG_UNASSIGNED;
  int64_t unassigned = n;
  int64_t* d = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  while (unassigned > 0) {
    int64_t nd = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (label[i] != AIRG_UNASSIGNED) continue;
      int maximal = 1;
      for (int64_t k = g->sym_rp[i]; k < g->sym_rp[i + 1]; ++k) {
        const int64_t j = g->sym_ci[k];
        if (label[j] == AIRG_UNASSIGNED && weight_less(w, i, j)) {
          maximal = 0;
          break;
        }
      }
      if (maximal) d[nd++] = i;
    }
    for (int64_t t = 0; t < nd; ++t) {
      label[d[t]] = AIRG_C;
      --unassigned;
    }
    for (int64_t t = 0; t < nd; ++t)
      for (int64_t k = g->sym_rp[d[t]]; k < g->sym_rp[d[t] + 1]; ++k) {
        const int64_t j = g->sym_ci[k];
        if (label[j] == AIRG_UNASSIGNED) {
          label[j] = AIRG_F;
          --unassigned;
        }
      }
  }
  if (swap)
    for (int64_t i = 0; i < n; ++i) label[i] = label[i] == AIRG_C ? AIRG_F : AIRG_C;
  free(d);
}

/* ------------------------------------------------------------------------ */
/* solve.cpp */
typedef struct {
  uint64_t fc, shadow;
} counters;

static double norm2(const double* v, int64_t n, counters* c) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += v[i] * v[i];
  if (c) c->fc += 2 * (uint64_t)n;
  return sqrt(acc);
}

/* coarse_solve solve.cpp:34-59 */
static void coarse_solve(const hier_t* h, const double* rhs, double* e, int64_t iters,
                         counters* c) {
  const int64_t n = h->coarse_a->n;
  double* r = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  double* ae = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  double* d = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    e[i] = 0.0;
    r[i] = rhs[i];
  }
  for (int64_t it = 0; it < iters; ++it) {
    if (it > 0) {
      spmv_into(h->coarse_a, e, ae);
      c->fc += 2 * (uint64_t)nnz_of(h->coarse_a);
      c->shadow += 2 * (uint64_t)nnz_of(h->coarse_a);
      for (int64_t i = 0; i < n; ++i) r[i] = rhs[i] - ae[i];
      c->fc += 2 * (uint64_t)n;
      c->shadow += 2 * (uint64_t)n;
    }
    spmv_into(h->coarse_inv, r, d);
    c->fc += 2 * (uint64_t)nnz_of(h->coarse_inv);
    c->shadow += 2 * (uint64_t)nnz_of(h->coarse_inv);
    for (int64_t i = 0; i < n; ++i) e[i] += 1.0 * d[i];
    c->fc += 2 * (uint64_t)n;
    c->shadow += 2 * (uint64_t)n;
  }
  free(r);
  free(ae);
  free(d);
}

/* f_smooth solve.cpp:63-87 */
static void f_smooth(const level_t* L, const double* b, double* x, counters* c) {
  const labelmap* map = &L->map;
  const int64_t nf = map->nf, ncc = map->nc;
  if (nf == 0) return;
  double* xf = (double*)xmalloc(sizeof(double) * (size_t)nf);
  double* xc = (double*)xmalloc(sizeof(double) * (size_t)(ncc ? ncc : 1));
  double* rf = (double*)xmalloc(sizeof(double) * (size_t)nf);
  double* afc = (double*)xmalloc(sizeof(double) * (size_t)nf);
  double* d = (double*)xmalloc(sizeof(double) * (size_t)nf);
  for (int64_t k = 0; k < nf; ++k) xf[k] = x[map->f_to_fine[k]];
  for (int64_t k = 0; k < ncc; ++k) xc[k] = x[map->c_to_fine[k]];
  spmv_into(L->aff, xf, rf);
  c->fc += 2 * (uint64_t)nnz_of(L->aff);
  spmv_into(L->afc, xc, afc);
  c->fc += 2 * (uint64_t)nnz_of(L->afc);
  c->shadow += 2 * (uint64_t)(nnz_of(L->aff) + nnz_of(L->afc));
  for (int64_t k = 0; k < nf; ++k) rf[k] = b[map->f_to_fine[k]] - rf[k] - afc[k];
  c->fc += 2 * (uint64_t)nf;
  c->shadow += 2 * (uint64_t)nf;
  spmv_into(L->ffinv, rf, d);
  c->fc += 2 * (uint64_t)nnz_of(L->ffinv);
  c->shadow += 2 * (uint64_t)nnz_of(L->ffinv);
  for (int64_t k = 0; k < nf; ++k) x[map->f_to_fine[k]] += d[k];
  c->fc += (uint64_t)nf;
  c->shadow += (uint64_t)nf;
  free(xf);
  free(xc);
  free(rf);
  free(afc);
  free(d);
}

/* vcycle_impl solve.cpp:93-146 with x_is_zero = true at entry (the only
 * way richardson_solve / vcycle / GMRES enter it with down_smooths = 0). */
static void vcycle_impl(const hier_t* h, int64_t l, const double* b, double* x, int x_is_zero,
                        const airg_solve_config* cfg, counters* c) {
  if (l == h->nlev) {
    const int64_t n = h->coarse_a->n;
    double* e = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
    if (x_is_zero) {
      coarse_solve(h, b, e, cfg->coarse_iterations, c);
      memcpy(x, e, sizeof(double) * (size_t)n);
    } else {
      double* r = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
      spmv_into(h->coarse_a, x, r);
      c->fc += 2 * (uint64_t)nnz_of(h->coarse_a);
      c->shadow += 2 * (uint64_t)nnz_of(h->coarse_a);
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
      c->fc += 2 * (uint64_t)n;
      c->shadow += 2 * (uint64_t)n;
      coarse_solve(h, r, e, cfg->coarse_iterations, c);
      for (int64_t i = 0; i < n; ++i) x[i] += 1.0 * e[i];
      c->fc += 2 * (uint64_t)n;
      c->shadow += 2 * (uint64_t)n;
      free(r);
    }
    free(e);
    return;
  }
  const level_t* L = &h->lev[l];
  const int64_t n = L->a->n, nc = L->map.nc;
  for (int64_t s = 0; s < cfg->down_smooths; ++s) {
    f_smooth(L, b, x, c);
    x_is_zero = 0;
  }
  double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
  if (x_is_zero) {
    memcpy(r, b, sizeof(double) * (size_t)n);
  } else {
    spmv_into(L->a, x, r);
    c->fc += 2 * (uint64_t)nnz_of(L->a);
    c->shadow += 2 * (uint64_t)nnz_of(L->a);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    c->fc += 2 * (uint64_t)n;
    c->shadow += 2 * (uint64_t)n;
  }
  double* rc = (double*)xmalloc(sizeof(double) * (size_t)(nc ? nc : 1));
  spmv_into(L->r, r, rc);
  c->fc += 2 * (uint64_t)nnz_of(L->r);
  c->shadow += 2 * (uint64_t)nnz_of(L->r);
  double* ec = (double*)xcalloc((size_t)(nc ? nc : 1), sizeof(double));
  vcycle_impl(h, l + 1, rc, ec, 1, cfg, c);
  double* pe = (double*)xmalloc(sizeof(double) * (size_t)n);
  spmv_into(L->p, ec, pe);
  c->fc += 2 * (uint64_t)nnz_of(L->p);
  c->shadow += 2 * (uint64_t)nnz_of(L->p);
  for (int64_t i = 0; i < n; ++i) x[i] += 1.0 * pe[i];
  c->fc += 2 * (uint64_t)n;
  c->shadow += 2 * (uint64_t)n;
  for (int64_t s = 0; s < cfg->up_f_smooths; ++s) f_smooth(L, b, x, c);
  free(r);
  free(rc);
  free(ec);
  free(pe);
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static const csr* top_of(const hier_t* h) { return h->nlev ? h->lev[0].a : h->coarse_a; }

/* richardson_solve solve.cpp:167-259 */
static void richardson(const hier_t* h, const double* b, const airg_solve_config* cfg, double* x,
                       airg_solve_stats* st, double* hist, int64_t cap) {
  const csr* a = top_of(h);
  const int64_t n = a->n;
  if (cfg->rtol <= 0.0) EINV("richardson_solve: rtol must be positive");
  counters c = {0, 0};
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  int64_t hl = 0;
#define PUSH(v)                     \
  do {                              \
    if (hist && hl < cap) hist[hl] = (v); \
    ++hl;                           \
  } while (0)
  const double t0 = now_s();
  const double bnorm = norm2(b, n, &c);
  c.shadow += 2 * (uint64_t)n;
  double* r = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  double* e = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  if (bnorm == 0.0) {
    st->converged = 1;
    PUSH(0.0);
  } else {
    for (int64_t it = 0;; ++it) {
      double rel;
      if (it == 0) {
        memcpy(r, b, sizeof(double) * (size_t)n);
        rel = 1.0;
      } else {
        spmv_into(a, x, e);
        c.fc += 2 * (uint64_t)nnz_of(a);
        c.shadow += 2 * (uint64_t)nnz_of(a);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - e[i];
        c.fc += 2 * (uint64_t)n;
        c.shadow += 2 * (uint64_t)n;
        rel = norm2(r, n, &c) / bnorm;
        c.shadow += 2 * (uint64_t)n;
      }
      PUSH(rel);
      st->final_relative_residual = rel;
      if (rel <= cfg->rtol) {
        st->converged = 1;
        st->iterations = it;
        break;
      }
      if (it >= cfg->max_iterations) {
        st->converged = 0;
        st->iterations = it;
        break;
      }
      for (int64_t i = 0; i < n; ++i) e[i] = 0.0;
      vcycle_impl(h, 0, r, e, 1, cfg, &c);
      for (int64_t i = 0; i < n; ++i) x[i] += 1.0 * e[i];
      c.fc += 2 * (uint64_t)n;
      c.shadow += 2 * (uint64_t)n;
    }
  }
  const double t1 = now_s();
  st->flops = c.fc;
  st->shadow_flops = c.shadow;
  st->work_units = (double)c.fc / (2.0 * (double)nnz_of(a));
  st->solve_seconds = t1 - t0;
  st->history_len = hl;
  free(r);
  free(e);
#undef PUSH
}

/* Outer right-preconditioned restarted GMRES (flexible storage Z = M V)
 * with classical Gram-Schmidt applied twice (CGS2) and Givens rotations.
 * NOT in the reference; the GPU implements the same steps
 * (paper_2408_08262_b200/csrc/solve.cu). One iteration = one Arnoldi step
 * = one V-cycle. Convergence is confirmed with a fresh matvec. */
static void gmres(const hier_t* h, const double* b, const airg_solve_config* cfg, double* x,
                  airg_solve_stats* st, double* hist, int64_t cap) {
  const csr* a = top_of(h);
  const int64_t n = a->n;
  const int64_t m = cfg->gmres_restart > 0 ? cfg->gmres_restart : 30;
  if (cfg->rtol <= 0.0) EINV("gmres_solve: rtol must be positive");
  counters c = {0, 0};
  int64_t hl = 0;
#define PUSH(v)                     \
  do {                              \
    if (hist && hl < cap) hist[hl] = (v); \
    ++hl;                           \
  } while (0)
  double* V = (double*)xmalloc(sizeof(double) * (size_t)(n * (m + 1) + 1));
  double* Z = (double*)xmalloc(sizeof(double) * (size_t)(n * m + 1));
  double* w = (double*)xmalloc(sizeof(double) * (size_t)(n + 1));
  double* r = (double*)xmalloc(sizeof(double) * (size_t)(n + 1));
  double* H = (double*)xcalloc((size_t)((m + 1) * m), sizeof(double));
  double *cs = (double*)xmalloc(sizeof(double) * (size_t)m),
         *sn = (double*)xmalloc(sizeof(double) * (size_t)m);
  double* g = (double*)xmalloc(sizeof(double) * (size_t)(m + 1));
  double* hcol = (double*)xmalloc(sizeof(double) * (size_t)(m + 1));
  double* y = (double*)xmalloc(sizeof(double) * (size_t)(m + 1));
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  const double t0 = now_s();
  const double bnorm = norm2(b, n, &c);
  int64_t its = 0;
  st->converged = 0;
  if (bnorm == 0.0) {
    st->converged = 1;
    PUSH(0.0);
    st->final_relative_residual = 0.0;
  } else {
    memcpy(r, b, sizeof(double) * (size_t)n);
    double beta = bnorm;
    PUSH(1.0);
    st->final_relative_residual = 1.0;
    while (its < cfg->max_iterations) {
      for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
      for (int64_t k = 0; k <= m; ++k) g[k] = 0.0;
      g[0] = beta;
      int64_t j = 0;
      for (; j < m && its < cfg->max_iterations; ++j) {
        double* vj = V + j * n;
        double* zj = Z + j * n;
        for (int64_t i = 0; i < n; ++i) zj[i] = 0.0;
        vcycle_impl(h, 0, vj, zj, 1, cfg, &c);
        spmv_into(a, zj, w);
        c.fc += 2 * (uint64_t)nnz_of(a);
        for (int64_t k = 0; k <= j; ++k) hcol[k] = 0.0;
        for (int pass = 0; pass < 2; ++pass) {
          double* dots = y; /* scratch, length >= j + 1 */
          for (int64_t k = 0; k <= j; ++k) {
            double s = 0.0;
            const double* vk = V + k * n;
            for (int64_t i = 0; i < n; ++i) s += vk[i] * w[i];
            dots[k] = s;
          }
          for (int64_t i = 0; i < n; ++i) {
            double s = w[i];
            for (int64_t k = 0; k <= j; ++k) s -= dots[k] * V[k * n + i];
            w[i] = s;
          }
          for (int64_t k = 0; k <= j; ++k) hcol[k] += dots[k];
          c.fc += 4 * (uint64_t)n * (uint64_t)(j + 1);
        }
        const double hn = norm2(w, n, &c);
        hcol[j + 1] = hn;
        double* vn = V + (j + 1) * n;
        for (int64_t i = 0; i < n; ++i) vn[i] = hn > 0.0 ? w[i] / hn : 0.0;
        for (int64_t k = 0; k < j; ++k) {
          const double t = cs[k] * hcol[k] + sn[k] * hcol[k + 1];
          hcol[k + 1] = -sn[k] * hcol[k] + cs[k] * hcol[k + 1];
          hcol[k] = t;
        }
        const double den = hypot(hcol[j], hcol[j + 1]);
        cs[j] = den > 0.0 ? hcol[j] / den : 1.0;
        sn[j] = den > 0.0 ? hcol[j + 1] / den : 0.0;
        hcol[j] = den;
        hcol[j + 1] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        for (int64_t k = 0; k <= j; ++k) H[k + j * (m + 1)] = hcol[k];
        ++its;
        const double est = fabs(g[j + 1]) / bnorm;
        PUSH(est);
        if (est <= cfg->rtol || hn == 0.0) {
          ++j;
          break;
        }
      }
      /* y = H(0:j,0:j) \ g(0:j); x += Z y */
      for (int64_t k = j - 1; k >= 0; --k) {
        double s = g[k];
        for (int64_t q = k + 1; q < j; ++q) s -= H[k + q * (m + 1)] * y[q];
        y[k] = s / H[k + k * (m + 1)];
      }
      for (int64_t i = 0; i < n; ++i) {
        double s = x[i];
        for (int64_t k = 0; k < j; ++k) s += y[k] * Z[k * n + i];
        x[i] = s;
      }
      spmv_into(a, x, w);
      c.fc += 2 * (uint64_t)nnz_of(a);
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - w[i];
      beta = norm2(r, n, &c);
      const double rel = beta / bnorm;
      st->final_relative_residual = rel;
      if (rel <= cfg->rtol) {
        st->converged = 1;
        break;
      }
      if (beta == 0.0) break;
    }
  }
  const double t1 = now_s();
  st->iterations = its;
  st->flops = c.fc;
  st->shadow_flops = c.fc;
  st->work_units = (double)c.fc / (2.0 * (double)nnz_of(a));
  st->solve_seconds = t1 - t0;
  st->history_len = hl;
  free(V);
  free(Z);
  free(w);
  free(r);
  free(H);
  free(cs);
  free(sn);
  free(g);
  free(hcol);
  free(y);
#undef PUSH
}

/* ======================================================================== */
/* exported API (same shapes as oracle/ref_capi.cpp) */

static csr* make_csr(int64_t n, int64_t m, const int64_t* rp, const int64_t* ci, const double* v) {
  csr* a = csr_new(n, m, rp[n]);
  memcpy(a->rp, rp, sizeof(int64_t) * (size_t)(n + 1));
  memcpy(a->ci, ci, sizeof(int64_t) * (size_t)rp[n]);
  memcpy(a->v, v, sizeof(double) * (size_t)rp[n]);
  csr_validate(a);
  return a;
}

int orc_mat_new(int64_t n, int64_t m, const int64_t* rp, const int64_t* ci, const double* v,
                void** out) {
  API_BEGIN
  *out = make_csr(n, m, rp, ci, v);
  API_END
}
int orc_mat_dims(const void* h, int64_t* n, int64_t* m, int64_t* nnz) {
  const csr* a = (const csr*)h;
  *n = a->n;
  *m = a->m;
  *nnz = nnz_of(a);
  return AIRG_OK;
}
int orc_mat_copy(const void* h, int64_t* rp, int64_t* ci, double* v) {
  const csr* a = (const csr*)h;
  memcpy(rp, a->rp, sizeof(int64_t) * (size_t)(a->n + 1));
  memcpy(ci, a->ci, sizeof(int64_t) * (size_t)nnz_of(a));
  memcpy(v, a->v, sizeof(double) * (size_t)nnz_of(a));
  return AIRG_OK;
}
int orc_mat_free(void* h) {
  csr_free((csr*)h);
  return AIRG_OK;
}
int orc_spmv(const void* a, const double* x, double* y) {
  spmv_into((const csr*)a, x, y);
  return AIRG_OK;
}
int orc_spgemm(const void* a, const void* b, void** out) {
  API_BEGIN
  *out = spgemm((const csr*)a, (const csr*)b);
  API_END
}
int orc_drop(const void* a, double tol, int keep, void** out) {
  API_BEGIN
  *out = drop_entries((const csr*)a, tol, keep);
  API_END
}
int orc_with_full_diagonal(const void* a, void** out) {
  API_BEGIN
  *out = with_full_diagonal((const csr*)a);
  API_END
}
int orc_extract_blocks(const void* a, const uint8_t* labels, void** aff, void** afc, void** acf) {
  API_BEGIN
  blocksplit s = extract_blocks((const csr*)a, labels);
  *aff = s.ff;
  *afc = s.fc;
  *acf = s.cf;
  csr_free(s.cc);
  map_free(&s.map);
  API_END
}
int orc_strength(const void* a, double alpha, void** s_out, int64_t* st_nnz) {
  API_BEGIN
  sgraph g = strength((const csr*)a, alpha);
  csr* s = csr_new(g.n, g.n, g.s_rp[g.n]);
  memcpy(s->rp, g.s_rp, sizeof(int64_t) * (size_t)(g.n + 1));
  memcpy(s->ci, g.s_ci, sizeof(int64_t) * (size_t)g.s_rp[g.n]);
  for (int64_t k = 0; k < g.s_rp[g.n]; ++k) s->v[k] = 1.0;
  if (st_nnz) *st_nnz = g.st_rp[g.n];
  graph_free(&g);
  *s_out = s;
  API_END
}
int orc_pmisr(const void* a, double alpha, int64_t max_loops, uint64_t seed, int32_t mode,
              uint8_t* labels, double* weights) {
  API_BEGIN
  sgraph g = strength((const csr*)a, alpha);
  double* w = make_weights(&g, seed, mode);
  pmisr_with_weights(&g, max_loops, w, labels);
  if (weights) memcpy(weights, w, sizeof(double) * (size_t)g.n);
  free(w);
  graph_free(&g);
  API_END
}
int orc_pmisr_with_weights(const void* s_pattern, int64_t max_loops, const double* w,
                           uint8_t* labels) {
  API_BEGIN
  const csr* s = (const csr*)s_pattern;
  sgraph g;
  memset(&g, 0, sizeof g);
  g.n = s->n;
  g.s_rp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(s->n + 1));
  g.s_ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(nnz_of(s) + 1));
  memcpy(g.s_rp, s->rp, sizeof(int64_t) * (size_t)(s->n + 1));
  memcpy(g.s_ci, s->ci, sizeof(int64_t) * (size_t)nnz_of(s));
  finish_graph(&g);
  pmisr_with_weights(&g, max_loops, w, labels);
  graph_free(&g);
  API_END
}
int orc_cf_split(const void* ap, double alpha, int64_t max_loops, uint64_t seed, int32_t mode,
                 int32_t ddc_enabled, double fraction, int64_t bins, uint8_t* labels,
                 uint8_t* labels_pre, airg_cf_report* rep) {
  API_BEGIN
  const csr* a = (const csr*)ap;
  sgraph g = strength(a, alpha);
  double* w = make_weights(&g, seed, mode);
  pmisr_with_weights(&g, max_loops, w, labels);
  free(w);
  memset(rep, 0, sizeof *rep);
  rep->s_nnz = g.s_rp[g.n];
  graph_free(&g);
  if (labels_pre) memcpy(labels_pre, labels, (size_t)a->n);
  blocksplit s = extract_blocks(a, labels);
  rep->n_f_pre = s.map.nf;
  if (ddc_enabled && s.map.nf > 0) {
    domrep dr;
    rep->n_converted = ddc(s.ff, labels, &s.map, fraction, bins, 0, 0.0, &dr);
    rep->max_theta = dr.max_theta;
    rep->alpha_diag = dr.alpha_diag;
    domrep_free(&dr);
  }
  split_free(&s);
  int64_t nf = 0;
  for (int64_t i = 0; i < a->n; ++i) nf += labels[i] == AIRG_F;
  rep->n_f = nf;
  rep->n_c = a->n - nf;
  API_END
}
int orc_ddc(const void* ap, uint8_t* labels, double fraction, int64_t bins, int32_t selection,
            double direct_alpha, airg_cf_report* rep) {
  API_BEGIN
  const csr* a = (const csr*)ap;
  blocksplit s = extract_blocks(a, labels);
  memset(rep, 0, sizeof *rep);
  rep->n_f_pre = s.map.nf;
  domrep dr;
  rep->n_converted = ddc(s.ff, labels, &s.map, fraction, bins, selection, direct_alpha, &dr);
  rep->max_theta = dr.max_theta;
  rep->alpha_diag = dr.alpha_diag;
  domrep_free(&dr);
  split_free(&s);
  API_END
}
int orc_poly_coefficients(const void* a, int64_t m, uint64_t seed, double* coeffs, int64_t* eff) {
  API_BEGIN
  compute_coefficients((const csr*)a, m, seed, coeffs, eff);
  API_END
}
int orc_poly_assemble(const void* a, const double* coeffs, int64_t nco, int64_t eff, int64_t s,
                      void** out) {
  API_BEGIN
  *out = assemble_fixed_sparsity((const csr*)a, coeffs, nco, eff, s, NULL);
  API_END
}
int orc_growth(const void* a, const void* q, double* out) {
  API_BEGIN
  *out = smoother_growth_estimate((const csr*)a, (const csr*)q);
  API_END
}
int orc_setup(const void* a, const airg_setup_config* cfg, void** out) {
  API_BEGIN
  *out = setup((const csr*)a, cfg);
  API_END
}
int orc_hier_free(void* h) {
  hier_destroy((hier_t*)h);
  return AIRG_OK;
}
int orc_hier_info(const void* hp, airg_hier_info* info) {
  const hier_t* h = (const hier_t*)hp;
  memset(info, 0, sizeof *info);
  info->n_levels = h->nlev;
  info->coarse_n = h->coarse_a->n;
  info->coarse_nnz = nnz_of(h->coarse_a);
  info->coarse_inv_nnz = nnz_of(h->coarse_inv);
  info->coarse_effective_order = h->coarse_eff;
  info->coarse_attempts = h->coarse_attempts;
  info->coarse_growth = h->coarse_growth;
  memcpy(info->coarse_coefficients, h->coarse_coeffs, sizeof(h->coarse_coeffs));
  info->grid_complexity = h->grid_c;
  info->operator_complexity = h->op_c;
  info->storage_complexity = h->store_c;
  return AIRG_OK;
}
int orc_level_info(const void* hp, int64_t l, airg_level_info* info) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  if (l < 0 || l >= h->nlev) EINV("level out of range");
  const level_t* L = &h->lev[l];
  memset(info, 0, sizeof *info);
  info->n = L->a->n;
  info->nnz = nnz_of(L->a);
  info->n_f = L->map.nf;
  info->n_c = L->map.nc;
  info->n_f_pre = L->n_f_pre;
  info->ddc_converted = L->n_converted;
  info->nnz_ff = nnz_of(L->aff);
  info->nnz_fc = nnz_of(L->afc);
  info->nnz_cf = nnz_of(L->acf);
  info->nnz_ffinv = nnz_of(L->ffinv);
  info->nnz_r = nnz_of(L->r);
  info->nnz_p = nnz_of(L->p);
  info->max_theta_pre = L->max_theta_pre;
  info->alpha_diag = L->alpha_diag;
  info->max_theta_post = L->max_theta_post;
  info->smoother_growth = L->growth;
  info->poly_attempts = L->attempts;
  info->effective_order = L->eff;
  memcpy(info->coefficients, L->coeffs, sizeof(L->coeffs));
  API_END
}
int orc_hier_matrix(const void* hp, int64_t l, int32_t which, const void** out) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  if (l == h->nlev) {
    if (which == 0)
      *out = h->coarse_a;
    else if (which == 4)
      *out = h->coarse_inv;
    else
      EINV("coarse level has only A (0) and inverse (4)");
  } else {
    if (l < 0 || l > h->nlev) EINV("level out of range");
    const level_t* L = &h->lev[l];
    const csr* m[7] = {L->a, L->aff, L->afc, L->acf, L->ffinv, L->r, L->p};
    if (which < 0 || which > 6) EINV("bad matrix selector");
    *out = m[which];
  }
  API_END
}
int orc_hier_labels(const void* hp, int64_t l, uint8_t* labels) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  if (l < 0 || l >= h->nlev) EINV("level out of range");
  memcpy(labels, h->lev[l].map.label, (size_t)h->lev[l].a->n);
  API_END
}
/* ---- single operations of the reference API (dominance_report, label map,
 * transfer operators, polynomial application, one F-smooth) ---- */
int orc_dominance_report(const void* aff, int64_t bins, double* theta, int64_t* hist, double* max_theta) {
  API_BEGIN
  domrep r = dominance_report((const csr*)aff, bins);
  if (theta) memcpy(theta, r.theta, sizeof(double) * (size_t)r.n);
  if (hist) memcpy(hist, r.hist, sizeof(int64_t) * (size_t)bins);
  if (max_theta) *max_theta = r.max_theta;
  domrep_free(&r);
  API_END
}
int orc_build_label_map(const uint8_t* labels, int64_t n, int64_t* fine_to_sub, int64_t* f_to_fine,
                        int64_t* c_to_fine, int64_t* n_f) {
  API_BEGIN
  labelmap m = build_label_map(labels, n);
  if (fine_to_sub) memcpy(fine_to_sub, m.fine_to_sub, sizeof(int64_t) * (size_t)n);
  if (f_to_fine) memcpy(f_to_fine, m.f_to_fine, sizeof(int64_t) * (size_t)m.nf);
  if (c_to_fine) memcpy(c_to_fine, m.c_to_fine, sizeof(int64_t) * (size_t)m.nc);
  if (n_f) *n_f = m.nf;
  map_free(&m);
  API_END
}
int orc_build_restriction(const void* acf, const void* ffinv, double drop, const uint8_t* labels, int64_t n,
                          void** out) {
  API_BEGIN
  labelmap m = build_label_map(labels, n);
  *out = build_restriction((const csr*)acf, (const csr*)ffinv, drop, &m);
  map_free(&m);
  API_END
}
int orc_build_prolongation(const void* ap, const void* s_pattern, const uint8_t* labels, void** out) {
  API_BEGIN
  const csr* a = (const csr*)ap;
  const csr* s = (const csr*)s_pattern;
  sgraph g;
  memset(&g, 0, sizeof g);
  g.n = s->n;
  g.s_rp = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(s->n + 1));
  g.s_ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(nnz_of(s) + 1));
  memcpy(g.s_rp, s->rp, sizeof(int64_t) * (size_t)(s->n + 1));
  memcpy(g.s_ci, s->ci, sizeof(int64_t) * (size_t)nnz_of(s));
  finish_graph(&g);
  labelmap m = build_label_map(labels, a->n);
  *out = build_prolongation(labels, &m, &g, a);
  map_free(&m);
  graph_free(&g);
  API_END
}
int orc_coarse_matrix(const void* r, const void* a, const void* p, double drop, void** out) {
  API_BEGIN
  *out = coarse_matrix((const csr*)r, (const csr*)a, (const csr*)p, drop);
  API_END
}
/* apply_polynomial gmres_poly.cpp:173-195: Horner, acc = c[deg] b, then
 * deg times acc = A acc; acc[i] += c[k] b[i] */
int orc_apply_polynomial(const void* ap, const double* coeffs, int64_t ncoeffs, int64_t deg, const double* b,
                         double* y) {
  API_BEGIN
  const csr* a = (const csr*)ap;
  if (ncoeffs < 1) EINV("apply_polynomial: empty polynomial");
  if (deg < 0 || deg >= ncoeffs) EINV("apply_polynomial: effective_order out of range");
  const int64_t n = a->n;
  double* acc = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  double* t = (double*)xmalloc(sizeof(double) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) acc[i] = coeffs[deg] * b[i];
  for (int64_t k = deg; k-- > 0;) {
    spmv_into(a, acc, t);
    const double alpha = coeffs[k];
    for (int64_t i = 0; i < n; ++i) acc[i] = t[i] + alpha * b[i];
  }
  memcpy(y, acc, sizeof(double) * (size_t)n);
  free(acc);
  free(t);
  API_END
}
int orc_f_smooth(const void* hp, int64_t l, const double* b, double* x) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  if (l < 0 || l >= h->nlev) EINV("f_smooth: level out of range");
  counters c = {0, 0};
  f_smooth(&h->lev[l], b, x, &c);
  API_END
}

int orc_vcycle(const void* hp, const airg_solve_config* cfg, const double* b, double* x) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  counters c = {0, 0};
  const int64_t n = top_of(h)->n;
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  vcycle_impl(h, 0, b, x, 1, cfg, &c);
  API_END
}
int orc_solve(const void* hp, const airg_solve_config* cfg, const double* b, double* x,
              airg_solve_stats* st, double* hist, int64_t cap) {
  API_BEGIN
  const hier_t* h = (const hier_t*)hp;
  memset(st, 0, sizeof *st);
  if (cfg->outer == 1)
    gmres(h, b, cfg, x, st, hist, cap);
  else
    richardson(h, b, cfg, x, st, hist, cap);
  st->grid_complexity = h->grid_c;
  st->operator_complexity = h->op_c;
  st->storage_complexity = h->store_c;
  API_END
}
