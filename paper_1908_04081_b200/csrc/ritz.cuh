// ritz.cuh -- Meurant-Tichy Ritz estimates (ritz.py:28-158) and Python's
// max/min semantics, shared by the s-step control kernel and HSCG.  Must be
// compiled with -fmad=false (build.py NO_FMAD): bit-exact with the reference.
#pragma once
#include <math.h>

#include "internal.cuh"

namespace {

// Python's max(a, b) / min(a, b) semantics (first argument wins unless the
// second compares strictly greater / smaller; NaN never compares)
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// ---------------------------------------------------------------------------
// Ritz estimates (ritz.py:28-158)
__device__ void ritz_init(RitzDev& r, double c0) {
  r.hi_om = 0.0; r.hi_h = 1.0; r.hi_zeta = 0.0; r.hi_init = 0;
  r.lo_om = 0.0; r.lo_a = 0.0; r.lo_d = 0.0; r.lo_g = 0.0; r.lo_h = 1.0; r.lo_init = 0;
  r.psi = 1.0; r.c = c0; r.eta_next = 0.0; r.count = 0; r.pad = 0;
}
__device__ __forceinline__ double ritz_lmax(const RitzDev& r) {
  return r.count >= 1 ? r.hi_om : (double)NAN;
}
__device__ __forceinline__ double ritz_lmin(const RitzDev& r) {
  return r.count >= 1 ? 1.0 / r.lo_om : (double)NAN;
}
__device__ bool ritz_absorb(RitzDev& r, double alpha, double beta) {
  if (!(alpha > 0.0 && beta > 0.0)) return false;  // BreakdownSignal, state untouched
  const double zeta = 1.0 / sqrt(alpha);
  const double eta = r.eta_next;
  if (!r.hi_init) {  // LmaxEstimator.absorb
    r.hi_om = zeta * zeta;
    r.hi_zeta = zeta;
    r.hi_init = 1;
  } else {
    const double le = r.hi_zeta * eta;
    const double d = (le * le) * r.hi_h;
    const double a = eta * eta + zeta * zeta;
    const double oa = r.hi_om - a;
    const double chi = sqrt(oa * oa + 4.0 * d);
    const double h = (chi != 0.0) ? 0.5 * (1.0 - oa / chi) : 0.0;
    r.hi_om = r.hi_om + chi * h;
    r.hi_h = h;
    r.hi_zeta = zeta;
  }
  if (!r.lo_init) {  // LminEstimator.absorb
    r.lo_om = 1.0 / (zeta * zeta);
    r.lo_a = r.lo_om;
    r.lo_init = 1;
  } else {
    const double dn = -(eta / zeta) * (r.lo_g * r.lo_d + r.lo_h * r.lo_a);
    const double an = (eta * eta * r.lo_a + 1.0) / (zeta * zeta);
    const double oa = r.lo_om - an;
    const double chi = sqrt(oa * oa + 4.0 * dn * dn);
    double h2;
    if (chi != 0.0) {
      h2 = 0.5 * (1.0 - oa / chi);
      h2 = py_max(h2, 0.0);
      h2 = py_min(h2, 1.0);
    } else {
      h2 = 0.0;
    }
    r.lo_om = r.lo_om + chi * h2;
    r.lo_g = sqrt(1.0 - h2);
    r.lo_h = copysign(sqrt(h2), dn);
    r.lo_d = dn;
    r.lo_a = an;
  }
  r.eta_next = sqrt(beta / alpha);
  r.psi = r.psi / (r.psi + beta);
  r.count += 1;
  if (r.count > 1) r.c = py_max(1.0, ritz_lmax(r) * sqrt(r.psi / ritz_lmin(r)));
  return true;
}
__device__ __forceinline__ double ritz_xi(const RitzDev& r) {
  if (r.count < 1) return 1.0;
  return py_max(1.0, ritz_lmax(r) * sqrt(r.psi / ritz_lmin(r)));
}

}  // namespace
