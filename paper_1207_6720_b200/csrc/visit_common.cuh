// visit_common.cuh -- host-side coefficient builders shared by the visit
// and staged-window smoother launchers.
#pragma once

#include <cmath>

#include "fmgsr_device.cuh"

namespace fmgsr {

template <typename T>
static GsCoef<T> make_coef(i64 n, double omega) {
  int k = level_of(n);
  GsCoef<T> g;
  double inv_h2 = pow4(k);
  g.inv_h2 = (T)inv_h2;
  g.rdiag = (T)(1.0 / (2.0 * inv_h2));  // exact power of two
  g.diag_b = (T)(3.0 * inv_h2);
  g.omega = (T)omega;
  g.diag_i = (T)(2.0 * inv_h2);
  return g;
}

template <typename T>
static KzCoef<T> make_kz(double pd) {
  KzCoef<T> k;
  int e;
  k.proj_diag = (T)pd;
  k.pow2 = std::frexp(pd, &e) == 0.5;  // pd = 2^(e-1): dividing is multiplying by 2^(1-e)
  k.recip = (T)(k.pow2 ? std::ldexp(1.0, 1 - e) : 1.0 / pd);
  return k;
}

}  // namespace fmgsr
