// The fast V-cycle's fused x-update kernel (solve.cu: one GPU; dist.cu: the
// row slabs), with a raw-pointer launcher.
#pragma once

#include "tiled.cuh"

namespace airg {
namespace {

// x_l = P e_c + [W r1 on the F rows] in one launch: blocks [0, bf) are lane
// groups over W's n_f rows, the rest one thread per C point (prolongation
// only). One-pass ascent (fused.cu): the same with K over e_c and y = W_k b_F
// from the descent (loaded with the row) in place of W over r1
// (ONEPASS: x_F = y + K e_c). When e_c was written two or more kernels back
// (EC_EARLY: the residual pass sits between), the prolongated values are
// loaded before the dependency wait; otherwise the predecessor is e_c's
// producer and they are read after it.
template <int G, bool ONEPASS, bool EC_EARLY>
__global__ void __launch_bounds__(kTileThreads)
k_fused_x(TileView w, int bf, const double* __restrict__ rv, const int32_t* __restrict__ f2f,
          const int32_t* __restrict__ c2f, int nc, const int32_t* __restrict__ pmap, const double* __restrict__ ec,
          double* __restrict__ x) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // every thread also prolongates C point t (C threads share the F rows'
  // blocks: fewer, fuller waves than separate C blocks)
  int ci = -1, cj = -1;
  double cv = 0.0;
  if (t < nc) {
    ci = __ldg(c2f + t);
    cj = __ldg(pmap + ci);
    if (EC_EARLY) cv = cj >= 0 ? ec[cj] : 0.0;
  }
  const int r = t / G, lane = t & (G - 1);
  const bool live = r < w.nrows;
  LaneRow<G, false> row;
  int i = 0, j = -1;
  double pe = 0.0;
  if (live) {
    row.load(w, r, lane);
    if (lane == 0) {
      i = __ldg(f2f + r);
      if (ONEPASS) {
        pe = rv[r];
      } else {
        j = __ldg(pmap + i);
        if (EC_EARLY) pe = j >= 0 ? ec[j] : 0.0;
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  if (!EC_EARLY) {
    if (ci >= 0) cv = cj >= 0 ? ec[cj] : 0.0;
    if (!ONEPASS && live && lane == 0) pe = j >= 0 ? ec[j] : 0.0;
  }
  double sf = 0.0, sc;
  if (live) row.dot(w, ONEPASS ? ec : rv, lane, sf, sc);
  sf = group_sum<G>(sf);
  if (live && lane == 0) x[i] = pe + sf;
  if (ci >= 0) x[ci] = cv;
}

// rv: r1 (or y with onepass); f2f / c2f: the F / C points' rows of x; pmap:
// the one-point map into ec's layout
inline void launch_fused_x_raw(Ctx& c, const Csr& m, const double* rv, const int32_t* f2f, const int32_t* c2f,
                               int nc, const int32_t* pmap, const double* ec, double* x, bool onepass,
                               bool ec_early) {
  const TileView w = tview(m);
  const int G = w.lanes;
  const int bf = (int)(((int64_t)w.nrows * G + kTileThreads - 1) / kTileThreads);
  const int bc = (nc + kTileThreads - 1) / kTileThreads;
  void (*k)(TileView, int, const double*, const int32_t*, const int32_t*, int, const int32_t*, const double*,
            double*) = nullptr;
#define AIRG_FX(O, E)                                                                                   \
  k = G == 1 ? &k_fused_x<1, O, E> : G == 2 ? &k_fused_x<2, O, E> : G == 4 ? &k_fused_x<4, O, E>          \
    : G == 8 ? &k_fused_x<8, O, E> : G == 16 ? &k_fused_x<16, O, E> : &k_fused_x<32, O, E>
  if (onepass)
    AIRG_FX(true, false);
  else if (ec_early)
    AIRG_FX(false, true);
  else
    AIRG_FX(false, false);
#undef AIRG_FX
  LAUNCH_PDL(c, k, (unsigned)std::max(1, std::max(bf, bc)), kTileThreads, 0, w, bf, rv, f2f, c2f, nc, pmap, ec, x);
}

}  // namespace
}  // namespace airg
