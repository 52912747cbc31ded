// Double-double arithmetic (host + device) for the GMRES-polynomial fit.
// The reference fits the polynomial in x87 long double (64-bit mantissa,
// gmres_poly.cpp:131-134); double-double (106-bit) is at least as accurate
// and exists on the GPU. Error-free transforms use explicit fma(), which
// --fmad=false leaves alone.
#pragma once
#include <cmath>

namespace airg {

struct dd {
  double hi, lo;
};

__host__ __device__ inline dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__host__ __device__ inline dd dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__host__ __device__ inline dd dd_add(dd x, dd y) {
  dd s = dd_two_sum(x.hi, y.hi);
  dd t = dd_two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__host__ __device__ inline dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__host__ __device__ inline dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__host__ __device__ inline dd dd_mul(dd x, dd y) {
  const double p = x.hi * y.hi;
  double e = fma(x.hi, y.hi, -p);
  e = fma(x.hi, y.lo, e);
  e = fma(x.lo, y.hi, e);
  return dd_quick(p, e);
}
__host__ __device__ inline dd dd_mul_d(dd x, double d) {
  const double p = x.hi * d;
  double e = fma(x.hi, d, -p);
  e = fma(x.lo, d, e);
  return dd_quick(p, e);
}
__host__ __device__ inline dd dd_from(double a) { return {a, 0.0}; }
__host__ __device__ inline dd dd_div(dd x, dd y) {
  const double q1 = x.hi / y.hi;
  dd r = dd_sub(x, dd_mul_d(y, q1));
  const double q2 = r.hi / y.hi;
  r = dd_sub(r, dd_mul_d(y, q2));
  const double q3 = r.hi / y.hi;
  dd q = dd_quick(q1, q2);
  return dd_add(q, dd_from(q3));
}
__host__ __device__ inline dd dd_sqrt(dd x) {
  if (x.hi <= 0.0) return {0.0, 0.0};
  const double s = sqrt(x.hi);
  // one Newton step: s + (x - s^2) / (2 s)
  const dd s2 = dd_mul(dd_from(s), dd_from(s));
  const dd r = dd_sub(x, s2);
  return dd_add(dd_from(s), dd_from(r.hi / (2.0 * s)));
}
__host__ __device__ inline double dd_abs_hi(dd x) { return fabs(x.hi); }

}  // namespace airg
