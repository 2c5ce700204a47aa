// kernels_ops.cu -- level operators and single-purpose kernels.
//
// Elementwise stencils over [n][ld] fields (block 32 x 8: lanes along the RHS
// columns, so each warp access is coalesced), the coarsest-level direct
// solve, the windowed Gauss-Seidel and Kaczmarz sweeps of the lane API, and
// the synthetic right-hand-side generators.  All arithmetic is exact-order
// (no contraction), matching the reference numpy/numba expressions cited.
#include <cmath>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

namespace {

constexpr int TX = 32, TY = 8;

inline dim3 grid_for(i64 rows, int B) {
  i64 gy = (rows + TY - 1) / TY;
  if (gy > 32768) gy = 32768;
  if (gy < 1) gy = 1;
  return dim3((unsigned)((B + TX - 1) / TX), (unsigned)gy);
}

#define ROWS_LOOP(i, rows) \
  for (i64 i = (i64)blockIdx.y * TY + threadIdx.y; i < (rows); i += (i64)gridDim.y * TY)

template <typename T>
__device__ __forceinline__ T inv_h2_of(i64 n) {
  int k = 0;
  while (((i64)1 << (k + 1)) <= n) k++;
  return (T)pow4(k);
}

// stencils.py:27-36
template <typename T>
__device__ __forceinline__ T lu_at(const T* u, i64 i, i64 n, i64 ld, T ih) {
  T s;
  if (i == 0) s = xsub(xmul(T(3), u[0]), u[ld]);
  else if (i == n - 1) s = xsub(xmul(T(3), u[(n - 1) * ld]), u[(n - 2) * ld]);
  else s = xsub(xsub(xmul(T(2), u[i * ld]), u[(i - 1) * ld]), u[(i + 1) * ld]);
  return xmul(s, ih);
}

template <typename T>
__device__ __forceinline__ T ru_at(const T* u, i64 j, i64 ld) {
  return xmul(T(0.5), xadd(u[(2 * j) * ld], u[(2 * j + 1) * ld]));
}

template <typename T>
__global__ void k_apply_operator(const T* __restrict__ u, T* __restrict__ out, i64 n, i64 ld, int B) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  T ih = inv_h2_of<T>(n);
  ROWS_LOOP(i, n) out[i * ld + r] = lu_at(u + r, i, n, ld, ih);
}

// stencils.py:39-47
template <typename T>
__global__ void k_restrict(const T* __restrict__ u, T* __restrict__ out, i64 nf, i64 ld, int B) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  ROWS_LOOP(j, nf / 2) out[j * ld + r] = ru_at(u + r, j, ld);
}

// stencils.py:50-64
template <typename T>
__device__ __forceinline__ T pc_at(const T* c, i64 i, i64 nc, i64 ld) {
  i64 nf = 2 * nc;
  if (i == 0) return xmul(T(0.5), c[0]);
  if (i == nf - 1) return xmul(T(0.5), c[(nc - 1) * ld]);
  if (i & 1) {
    i64 j = (i - 1) / 2;
    return xmul(T(0.25), xadd(xmul(T(3), c[j * ld]), c[(j + 1) * ld]));
  }
  i64 j = (i - 2) / 2;
  return xmul(T(0.25), xadd(c[j * ld], xmul(T(3), c[(j + 1) * ld])));
}

template <typename T>
__global__ void k_prolong_correction(const T* __restrict__ c, T* __restrict__ out, i64 nc, i64 ld,
                                     int B) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  ROWS_LOOP(i, 2 * nc) out[i * ld + r] = pc_at(c + r, i, nc, ld);
}

// stencils.py:67-105 (one fine row)
template <typename T>
__device__ __forceinline__ T pf_at(const T* c, i64 i, i64 n, i64 ld) {
  i64 nf = 2 * n;
#define C(k) c[(k) * ld]
  T v;
  if (i == 0) v = xsub(xmul(T(70), C(0)), xmul(T(2), C(1)));
  else if (i == 1) v = xsub(xadd(xmul(T(112), C(0)), xmul(T(35), C(1))), xmul(T(5), C(2)));
  else if (i == 2) v = xsub(xadd(xmul(T(40), C(0)), xmul(T(105), C(1))), xmul(T(7), C(2)));
  else if (i == 3)
    v = xsub(xadd(xadd(xmul(T(-7), C(0)), xmul(T(105), C(1))), xmul(T(35), C(2))), xmul(T(5), C(3)));
  else if (i == nf - 4)
    v = xsub(xadd(xadd(xmul(T(-7), C(n - 1)), xmul(T(105), C(n - 2))), xmul(T(35), C(n - 3))),
             xmul(T(5), C(n - 4)));
  else if (i == nf - 3)
    v = xsub(xadd(xmul(T(40), C(n - 1)), xmul(T(105), C(n - 2))), xmul(T(7), C(n - 3)));
  else if (i == nf - 2)
    v = xsub(xadd(xmul(T(112), C(n - 1)), xmul(T(35), C(n - 2))), xmul(T(5), C(n - 3)));
  else if (i == nf - 1) v = xsub(xmul(T(70), C(n - 1)), xmul(T(2), C(n - 2)));
  else if ((i & 1) == 0) {
    i64 q = i / 2;
    v = xsub(xadd(xadd(xmul(T(-5), C(q - 2)), xmul(T(35), C(q - 1))), xmul(T(105), C(q))),
             xmul(T(7), C(q + 1)));
  } else {
    i64 q = (i - 1) / 2;
    v = xsub(xadd(xadd(xmul(T(-7), C(q - 1)), xmul(T(105), C(q))), xmul(T(35), C(q + 1))),
             xmul(T(5), C(q + 2)));
  }
#undef C
  return xdiv(v, T(128));
}

template <typename T>
__global__ void k_prolong_fmg(const T* __restrict__ c, T* __restrict__ out, i64 nc, i64 ld, int B) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  ROWS_LOOP(i, 2 * nc) out[i * ld + r] = pf_at(c + r, i, nc, ld);
}

// stencils.py:108-125.  mode 0: tau; 1: coarse_rhs; 2: restrict + coarse_rhs.
template <typename T>
__global__ void k_restrict_tau(const T* __restrict__ u, const T* __restrict__ f, T* __restrict__ uH,
                               T* __restrict__ fH, i64 nf, i64 ld, int B, int mode, bool nl) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  const i64 nc = nf / 2;
  const T ih = inv_h2_of<T>(nf), iH = inv_h2_of<T>(nc);
  const T* ur = u + r;
  ROWS_LOOP(j, nc) {
    T Rj = ru_at(ur, j, ld);
    T LH;
    if (j == 0) LH = xmul(xsub(xmul(T(3), Rj), ru_at(ur, 1, ld)), iH);
    else if (j == nc - 1) LH = xmul(xsub(xmul(T(3), Rj), ru_at(ur, nc - 2, ld)), iH);
    else LH = xmul(xsub(xsub(xmul(T(2), Rj), ru_at(ur, j - 1, ld)), ru_at(ur, j + 1, ld)), iH);
    T L0 = lu_at(ur, 2 * j, nf, ld, ih), L1 = lu_at(ur, 2 * j + 1, nf, ld, ih);
    if (nl) {  // N(u) = L u + u^3 on both levels (orc_coarse_rhs_nl)
      T a = ur[(2 * j) * ld], b = ur[(2 * j + 1) * ld];
      L0 = xadd(L0, xmul(xmul(a, a), a));
      L1 = xadd(L1, xmul(xmul(b, b), b));
      LH = xadd(LH, xmul(xmul(Rj, Rj), Rj));
    }
    T RL = xmul(T(0.5), xadd(L0, L1));
    T tau = xsub(LH, RL);
    if (mode == 0) {
      fH[j * ld + r] = tau;
    } else {
      T Rf = ru_at(f + r, j, ld);
      fH[j * ld + r] = xadd(Rf, tau);
      if (mode == 2) uH[j * ld + r] = Rj;
    }
  }
}

// The same restriction + tau as a streaming pass: each thread walks a segment
// of coarse rows of one column with a sliding window (pair j-1, j, j+1), so
// every fine row is loaded once.  Bitwise the expressions of k_restrict_tau.
template <typename T, bool NL>
__global__ void __launch_bounds__(256) k_restrict_tau_seg(const T* __restrict__ u,
                                                          const T* __restrict__ f,
                                                          T* __restrict__ uH, T* __restrict__ fH,
                                                          i64 nf, i64 ld, int B, int mode, i64 seg) {
  const int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  const i64 nc = nf / 2;
  const i64 j0 = ((i64)blockIdx.y * blockDim.y + threadIdx.y) * seg;
  if (j0 >= nc) return;
  const i64 j1 = j0 + seg < nc ? j0 + seg : nc;
  const T ih = inv_h2_of<T>(nf), iH = inv_h2_of<T>(nc);
  const T* ur = u + r;
  const T* fr = f + r;
  T m1 = T(0), Rm = T(0);  // u[2j-1], R u at j-1
  if (j0 > 0) {
    T a = __ldg(ur + (2 * j0 - 2) * ld);
    m1 = __ldg(ur + (2 * j0 - 1) * ld);
    Rm = xmul(T(0.5), xadd(a, m1));
  }
  T c0 = __ldg(ur + (2 * j0) * ld), c1 = __ldg(ur + (2 * j0 + 1) * ld);
  T Rc = xmul(T(0.5), xadd(c0, c1));
  constexpr int K = 4;  // coarse rows per batch: all loads of a batch issued first
  for (i64 jb = j0; jb < j1; jb += K) {
    T un[2 * K], fv[2 * K];
#pragma unroll
    for (int k = 0; k < 2 * K; k++) {
      i64 iu = 2 * jb + 2 + k, iv = 2 * jb + k;
      un[k] = __ldg(ur + (iu < nf ? iu : nf - 1) * ld);
      fv[k] = mode ? __ldg(fr + (iv < nf ? iv : nf - 1) * ld) : T(0);
    }
#pragma unroll
    for (int k = 0; k < K; k++) {
      const i64 j = jb + k;
      if (j >= j1) break;
      T n0 = T(0), n1 = T(0), Rn = T(0);
      if (j + 1 < nc) {
        n0 = un[2 * k];
        n1 = un[2 * k + 1];
        Rn = xmul(T(0.5), xadd(n0, n1));
      }
      T LH;
      if (j == 0) LH = xmul(xsub(xmul(T(3), Rc), Rn), iH);
      else if (j == nc - 1) LH = xmul(xsub(xmul(T(3), Rc), Rm), iH);
      else LH = xmul(xsub(xsub(xmul(T(2), Rc), Rm), Rn), iH);
      T L0 = (j == 0) ? xmul(xsub(xmul(T(3), c0), c1), ih)
                      : xmul(xsub(xsub(xmul(T(2), c0), m1), c1), ih);
      T L1 = (j == nc - 1) ? xmul(xsub(xmul(T(3), c1), c0), ih)
                           : xmul(xsub(xsub(xmul(T(2), c1), c0), n0), ih);
      if (NL) {
        L0 = xadd(L0, xmul(xmul(c0, c0), c0));
        L1 = xadd(L1, xmul(xmul(c1, c1), c1));
        LH = xadd(LH, xmul(xmul(Rc, Rc), Rc));
      }
      T tau = xsub(LH, xmul(T(0.5), xadd(L0, L1)));
      if (mode == 0) {
        fH[j * ld + r] = tau;
      } else {
        T Rf = xmul(T(0.5), xadd(fv[2 * k], fv[2 * k + 1]));
        fH[j * ld + r] = xadd(Rf, tau);
        if (mode == 2) uH[j * ld + r] = Rc;
      }
      m1 = c1;
      Rm = Rc;
      c0 = n0;
      c1 = n1;
      Rc = Rn;
    }
  }
}

// cycles.py:120-121: out = u + prolong_correction(uH - restrict(u))
template <typename T>
__global__ void k_fas_correct(const T* __restrict__ u, const T* __restrict__ uH, T* __restrict__ out,
                              i64 nf, i64 ld, int B) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  const i64 nc = nf / 2;
  const T* ur = u + r;
  const T* hr = uH + r;
  ROWS_LOOP(i, nf) {
    auto c = [&](i64 j) { return xsub(hr[j * ld], ru_at(ur, j, ld)); };
    T p;
    if (i == 0) p = xmul(T(0.5), c(0));
    else if (i == nf - 1) p = xmul(T(0.5), c(nc - 1));
    else if (i & 1) {
      i64 j = (i - 1) / 2;
      p = xmul(T(0.25), xadd(xmul(T(3), c(j)), c(j + 1)));
    } else {
      i64 j = (i - 2) / 2;
      p = xmul(T(0.25), xadd(c(j), xmul(T(3), c(j + 1))));
    }
    out[i * ld + r] = xadd(ur[i * ld], p);
  }
}

// smoothers.py:210-225 -> scipy solveh_banded -> LAPACK ?ptsv: dpttrf (L D L^T)
// then dptts2.  The factor depends on n only; pt_factor builds it with the
// dpttrf operation order (into shared memory per block, or once into a global
// workspace for large n); pt_solve runs dptts2, one thread per RHS.
template <typename T>
__device__ void pt_factor(T* d, T* e, i64 n) {
  T ih = inv_h2_of<T>(n);
  for (i64 i = 0; i < n; i++) d[i] = xmul(T(2), ih);
  d[0] = xmul(T(3), ih);
  d[n - 1] = xmul(T(3), ih);
  for (i64 i = 0; i < n - 1; i++) e[i] = -ih;
  for (i64 i = 0; i < n - 1; i++) {
    T ei = e[i];
    e[i] = xdiv(ei, d[i]);
    d[i + 1] = xsub(d[i + 1], xmul(e[i], ei));
  }
}

template <typename T>
__global__ void k_pt_factor(T* fac, i64 n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) pt_factor(fac, fac + n, n);
}

template <typename T>
__global__ void k_direct_solve(const T* __restrict__ f, T* __restrict__ u, i64 n, i64 ld, int B,
                               const T* __restrict__ fac) {
  extern __shared__ unsigned char smem_raw[];
  const T* d;
  const T* e;
  if (fac) {
    d = fac;
    e = fac + n;
  } else {
    T* ds = reinterpret_cast<T*>(smem_raw);
    if (threadIdx.x == 0) pt_factor(ds, ds + n, n);
    __syncthreads();
    d = ds;
    e = ds + n;
  }
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const T* fr = f + r;
  T* ur = u + r;
  T prev = fr[0];
  ur[0] = prev;
  for (i64 i = 1; i < n; i++) {
    prev = xsub(fr[i * ld], xmul(prev, e[i - 1]));
    ur[i * ld] = prev;
  }
  T nxt = xdiv(prev, d[n - 1]);
  ur[(n - 1) * ld] = nxt;
  for (i64 i = n - 2; i >= 0; i--) {
    nxt = xsub(xdiv(ur[i * ld], d[i]), xmul(nxt, e[i]));
    ur[i * ld] = nxt;
  }
}

// problem.py:61-77 direct_fine_solve -> scipy solve_banded((1, 1), ab, f) ->
// LAPACK dgbsv: dgbtf2 (LU with partial pivoting; multipliers are the
// sub-diagonal scaled by RN(1/pivot) as DSCAL does; the trailing update is the
// DGER rank-1 step a + l * (-(super))), then dgbtrs (the DGER forward sweep
// b_{j+1} + l_j * (-b_j), skipped when b_j == 0, and DTBSV's upper back
// substitution over the KL + KU = 2 superdiagonals, the second being the
// zero fill-in).  An algorithm independent of the L D L^T coarse solve above,
// as the reference intends ("general LU here, Cholesky there").  This
// operator is strictly diagonally dominant after the first column, so the
// pivot search never swaps rows; the factor kernel checks that and flags it.
template <typename T>
__global__ void k_gb_factor(T* fac, i64 n, int* bad) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const T ih = inv_h2_of<T>(n);
  T* u = fac;      // pivots u_jj
  T* l = fac + n;  // multipliers l_j (row j+1 of column j)
  T dj = xmul(T(3), ih);
  int swaps = 0;
  for (i64 j = 0; j < n; j++) {
    u[j] = dj;
    if (j == n - 1) break;
    const T sub = -ih;
    if (fabs(sub) > fabs(dj)) swaps++;  // IDAMAX would pick the sub-diagonal
    const T lj = xmul(xrcp(dj), sub);   // DSCAL(1, ONE / AB(KV+1, J), ...)
    l[j] = lj;
    const T temp = -sub;                // DGER: TEMP = -ONE * A(J, J+1)
    const T a = (j + 1 == n - 1) ? xmul(T(3), ih) : xmul(T(2), ih);
    dj = xadd(a, xmul(lj, temp));
  }
  if (swaps) atomicAdd(bad, swaps);
}

template <typename T>
__global__ void k_gb_solve(const T* __restrict__ f, T* __restrict__ x, i64 n, i64 ld, int B,
                           const T* __restrict__ fac) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const T ih = inv_h2_of<T>(n);
  const T* u = fac;
  const T* l = fac + n;
  const T* fr = f + r;
  T* xr = x + r;
  // dgbtrs forward: DGER(1, NRHS, -ONE, l_j, 1, B(J, :), LDB, B(J+1, :), LDB)
  T prev = fr[0];
  xr[0] = prev;
  for (i64 j = 0; j + 1 < n; j++) {
    T b = fr[(j + 1) * ld];
    if (prev != T(0)) b = xadd(b, xmul(l[j], -prev));
    xr[(j + 1) * ld] = b;
    prev = b;
  }
  // DTBSV('U', 'N', 'N', n, 2, AB, LDAB, x): column-oriented back substitution;
  // c0 = x_j (final input), c1 = x_{j-1} (after step j+1's update)
  const T sup = -ih;
  T c0 = prev;
  T c1 = n >= 2 ? xr[(n - 2) * ld] : T(0);
  for (i64 j = n - 1; j >= 0; j--) {
    T c2 = j >= 2 ? xr[(j - 2) * ld] : T(0);
    if (c0 != T(0)) {
      c0 = xdiv(c0, u[j]);
      c1 = xsub(c1, xmul(c0, sup));
      c2 = xsub(c2, xmul(c0, T(0)));  // the zero fill-in row of the band
    }
    xr[j * ld] = c0;
    c0 = c1;
    c1 = c2;
  }
}

// _kernels_numba.py:15-36, one thread per RHS, in place
template <typename T>
__global__ void k_gs_sweep(T* u, const T* __restrict__ f, i64 n, i64 ld, int B, GsCoef<T> gc,
                           i64 start, i64 stop, bool forward) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  T* ur = u + r;
  const T* fr = f + r;
  if (forward) {
    T uL = start > 0 ? ur[(start - 1) * ld] : T(0);
    T cur = ur[start * ld];
    for (i64 i = start; i < stop; i++) {
      T nxt = (i + 1 < n) ? ur[(i + 1) * ld] : T(0);
      T v = gs_cell(gc, i, n, uL, cur, nxt, fr[i * ld]);
      ur[i * ld] = v;
      uL = v;
      cur = nxt;
    }
  } else {
    T uR = stop < n ? ur[stop * ld] : T(0);
    T cur = ur[(stop - 1) * ld];
    for (i64 i = stop - 1; i >= start; i--) {
      T prv = i > 0 ? ur[(i - 1) * ld] : T(0);
      T v = gs_cell(gc, i, n, prv, cur, uR, fr[i * ld]);
      ur[i * ld] = v;
      uR = v;
      cur = prv;
    }
  }
}

// _kernels_numba.py:39-57: disjoint pairs, so every pair is projected
// independently (the sweep direction cannot change the result).
template <typename T>
__global__ void k_kaczmarz(T* u, const T* __restrict__ uc, i64 j0, i64 j1, i64 ld, int B,
                           KzCoef<T> kz) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  ROWS_LOOP(k, j1 - j0) {
    i64 j = j0 + k;
    T a = u[(2 * j) * ld + r], b = u[(2 * j + 1) * ld + r];
    kaczmarz_pair(a, b, uc[j * ld + r], kz);
    u[(2 * j) * ld + r] = a;
    u[(2 * j + 1) * ld + r] = b;
  }
}

// Synthetic Fourier forcing: f = sum_k a_k sin(k pi x),
// u* = sum_k a_k sin(k pi x) / (k pi)^2, x_i = (i + 1/2)/n; coef is [B][K].
template <typename T>
__global__ void k_fourier_rhs(const double* __restrict__ coef, int K, i64 n, i64 ld, int B, T* f,
                              T* uex) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  const double* a = coef + (i64)r * K;
  ROWS_LOOP(i, n) {
    double x = ((double)i + 0.5) / (double)n;
    double fs = 0.0, us = 0.0;
    for (int k = 1; k <= K; k++) {
      double s = sinpi((double)k * x);
      double kp = (double)k * M_PI;
      fs += a[k - 1] * s;
      us += a[k - 1] * s / (kp * kp);
    }
    f[i * ld + r] = (T)fs;
    if (uex) uex[i * ld + r] = (T)us;
  }
}

// The study harness's manufactured problem (reference problem.py:23-46):
// f = sum over odd j <= K of sin(j pi x)/j, u = sum sin(j pi x)/(j (j pi)^2),
// one thread per cell (a single right-hand side, ld = 1).
__global__ void k_manufactured(i64 n, i64 K, double* f, double* uex) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const double x = ((double)i + 0.5) / (double)n;
    double fs = 0.0, us = 0.0;
    for (i64 j = 1; j <= K; j += 2) {
      const double s = sinpi((double)j * x);
      const double jp = (double)j * M_PI;
      fs += s / (double)j;
      us += s / ((double)j * (jp * jp));
    }
    f[i] = fs;
    if (uex) uex[i] = us;
  }
}

// Nonlinear manufactured problem (BASELINE config 3): u = s x(1-x)e^x,
// f = s x(x+3)e^x + (s x(1-x)e^x)^3 for -u'' + u^3 = f.
template <typename T>
__global__ void k_nonlinear_rhs(const double* __restrict__ scale, i64 n, i64 ld, int B, T* f,
                                T* uex) {
  int r = blockIdx.x * TX + threadIdx.x;
  if (r >= B) return;
  const double s = scale[r];
  ROWS_LOOP(i, n) {
    double x = ((double)i + 0.5) / (double)n;
    double ex = exp(x);
    double u = s * x * (1.0 - x) * ex;
    f[i * ld + r] = (T)(s * x * (x + 3.0) * ex + u * u * u);
    if (uex) uex[i * ld + r] = (T)u;
  }
}

}  // namespace

void launch_manufactured(i64 n, i64 K, double* f, double* uex, cudaStream_t s) {
  require(n >= 1 && K >= 1 && f, "manufactured_rhs: bad arguments");
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_manufactured<<<(unsigned)blocks, 256, 0, s>>>(n, K, f, uex);
  check_launch("manufactured_rhs");
}


template <typename T>
void launch_apply_operator(const T* u, T* out, i64 n, i64 ld, int B, cudaStream_t s) {
  require(n >= 2 && is_pow2(n), "apply_operator: size must be a power of two >= 2");
  k_apply_operator<T><<<grid_for(n, B), dim3(TX, TY), 0, s>>>(u, out, n, ld, B);
  check_launch("apply_operator");
}
template <typename T>
void launch_restrict(const T* u, T* out, i64 nf, i64 ld, int B, cudaStream_t s) {
  require(nf >= 2 && is_pow2(nf), "restrict: size must be a power of two >= 2");
  k_restrict<T><<<grid_for(nf / 2, B), dim3(TX, TY), 0, s>>>(u, out, nf, ld, B);
  check_launch("restrict");
}
template <typename T>
void launch_prolong_correction(const T* c, T* out, i64 nc, i64 ld, int B, cudaStream_t s) {
  require(nc >= 2 && is_pow2(nc), "prolong_correction: size must be a power of two >= 2");
  k_prolong_correction<T><<<grid_for(2 * nc, B), dim3(TX, TY), 0, s>>>(c, out, nc, ld, B);
  check_launch("prolong_correction");
}
template <typename T>
void launch_prolong_fmg(const T* c, T* out, i64 nc, i64 ld, int B, cudaStream_t s) {
  require(nc >= 4 && is_pow2(nc), "prolong_fmg: coarse size must be a power of two >= 4");
  k_prolong_fmg<T><<<grid_for(2 * nc, B), dim3(TX, TY), 0, s>>>(c, out, nc, ld, B);
  check_launch("prolong_fmg");
}
template <typename T>
void launch_restrict_tau(const T* u, const T* f, T* uH, T* fH, i64 nf, i64 ld, int B, int mode,
                         cudaStream_t s, bool nl) {
  require(nf >= 4 && is_pow2(nf), "tau: fine size must be a power of two >= 4");
  // segments sized for ~2 resident waves of 256-thread blocks on 148 SMs
  const i64 nc = nf / 2;
  const i64 cols = (i64)((B + TX - 1) / TX) * TX;
  i64 nseg = (148 * 2048) / cols;
  if (nseg < 1) nseg = 1;
  i64 seg = (nc + nseg - 1) / nseg;
  if (seg < 8) seg = 8;
  nseg = (nc + seg - 1) / seg;
  dim3 grid((unsigned)((B + TX - 1) / TX), (unsigned)((nseg + TY - 1) / TY));
  if (nl) k_restrict_tau_seg<T, true><<<grid, dim3(TX, TY), 0, s>>>(u, f, uH, fH, nf, ld, B, mode, seg);
  else k_restrict_tau_seg<T, false><<<grid, dim3(TX, TY), 0, s>>>(u, f, uH, fH, nf, ld, B, mode, seg);
  check_launch("restrict_tau");
}

// Newton solve of N(u) = L u + u^3 = f (orc_direct_solve_nl): linear solve as
// the first iterate, then NEWTON_STEPS steps, each a tridiagonal L + diag(3u^2)
// solve in the dpttrf / dptts2 order.  One thread per RHS; u lives in the
// output column, the factor and residual in per-thread local arrays.
constexpr int NEWTON_STEPS = 10;
constexpr int NEWTON_NMAX = 64;

template <typename T>
__global__ void k_direct_solve_nl(const T* __restrict__ f, T* __restrict__ u, i64 n, i64 ld, int B) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  T d[NEWTON_NMAX], e[NEWTON_NMAX], rr[NEWTON_NMAX];
  const T ih = inv_h2_of<T>(n);
  const T* fr = f + r;
  T* ur = u + r;
  // linear first iterate (k_direct_solve)
  pt_factor(d, e, n);
  T prev = fr[0];
  ur[0] = prev;
  for (i64 i = 1; i < n; i++) {
    prev = xsub(fr[i * ld], xmul(prev, e[i - 1]));
    ur[i * ld] = prev;
  }
  T nx = xdiv(prev, d[n - 1]);
  ur[(n - 1) * ld] = nx;
  for (i64 i = n - 2; i >= 0; i--) {
    nx = xsub(xdiv(ur[i * ld], d[i]), xmul(nx, e[i]));
    ur[i * ld] = nx;
  }
  for (int it = 0; it < NEWTON_STEPS; it++) {
    for (i64 i = 0; i < n; i++) {
      T ui = ur[i * ld];
      T Ni = xadd(lu_at(ur, i, n, ld, ih), xmul(xmul(ui, ui), ui));
      rr[i] = xsub(fr[i * ld], Ni);
      d[i] = xadd(xmul(T((i == 0 || i == n - 1) ? 3 : 2), ih), xmul(T(3), xmul(ui, ui)));
      e[i] = -ih;
    }
    for (i64 i = 0; i < n - 1; i++) {
      T ei = e[i];
      e[i] = xdiv(ei, d[i]);
      d[i + 1] = xsub(d[i + 1], xmul(e[i], ei));
    }
    for (i64 i = 1; i < n; i++) rr[i] = xsub(rr[i], xmul(rr[i - 1], e[i - 1]));
    rr[n - 1] = xdiv(rr[n - 1], d[n - 1]);
    for (i64 i = n - 2; i >= 0; i--) rr[i] = xsub(xdiv(rr[i], d[i]), xmul(rr[i + 1], e[i]));
    for (i64 i = 0; i < n; i++) ur[i * ld] = xadd(ur[i * ld], rr[i]);
  }
}

template <typename T>
void launch_direct_solve_nl(const T* f, T* u, i64 n, i64 ld, int B, cudaStream_t s) {
  require(n >= 2 && is_pow2(n) && n <= NEWTON_NMAX, "nonlinear direct solve: n must be a power of two in [2, 64]");
  k_direct_solve_nl<T><<<(B + 127) / 128, 128, 0, s>>>(f, u, n, ld, B);
  check_launch("direct_solve_nl");
}
template <typename T>
void launch_fas_correct(const T* u, const T* uH, T* out, i64 nf, i64 ld, int B, cudaStream_t s) {
  require(nf >= 4 && is_pow2(nf), "fas_correct: fine size must be a power of two >= 4");
  k_fas_correct<T><<<grid_for(nf, B), dim3(TX, TY), 0, s>>>(u, uH, out, nf, ld, B);
  check_launch("fas_correct");
}
template <typename T>
void launch_direct_solve(const T* f, T* u, i64 n, i64 ld, int B, cudaStream_t s, T* workspace) {
  require(n >= 2 && is_pow2(n), "direct_solve: size must be a power of two >= 2");
  int threads = 128;
  if (workspace) {
    k_pt_factor<T><<<1, 1, 0, s>>>(workspace, n);
    check_launch("pt_factor");
    k_direct_solve<T><<<(B + threads - 1) / threads, threads, 0, s>>>(f, u, n, ld, B, workspace);
  } else {
    require(n <= 2048, "direct_solve: n > 2048 needs a workspace of 2n elements");
    size_t smem = 2 * (size_t)n * sizeof(T);
    k_direct_solve<T><<<(B + threads - 1) / threads, threads, smem, s>>>(f, u, n, ld, B, nullptr);
  }
  check_launch("direct_solve");
}
template <typename T>
void launch_banded_lu_solve(const T* f, T* u, i64 n, i64 ld, int B, T* workspace, int* bad,
                            cudaStream_t s) {
  require(n >= 2 && is_pow2(n), "banded_lu_solve: size must be a power of two >= 2");
  require(workspace != nullptr && bad != nullptr, "banded_lu_solve: null workspace");
  k_gb_factor<T><<<1, 1, 0, s>>>(workspace, n, bad);
  check_launch("gb_factor");
  k_gb_solve<T><<<(B + 127) / 128, 128, 0, s>>>(f, u, n, ld, B, workspace);
  check_launch("gb_solve");
}
template <typename T>
void launch_gs_sweep(T* u, const T* f, i64 n, i64 ld, int B, double inv_h2, i64 start, i64 stop,
                     bool forward, double omega, cudaStream_t s) {
  require(0 <= start && start < stop && stop <= n, "gs_sweep: window outside [0, n)");
  GsCoef<T> gc;
  gc.inv_h2 = (T)inv_h2;
  gc.rdiag = (T)(1.0 / (2.0 * inv_h2));
  gc.diag_b = (T)(3.0 * inv_h2);
  gc.omega = (T)omega;
  gc.diag_i = (T)(2.0 * inv_h2);
  // rdiag must be exact: inv_h2 a power of two (true for every level, 4^k)
  int e;
  require(std::frexp(inv_h2, &e) == 0.5, "gs_sweep: inv_h2 must be a power of two");
  k_gs_sweep<T><<<(B + 127) / 128, 128, 0, s>>>(u, f, n, ld, B, gc, start, stop, forward);
  check_launch("gs_sweep");
}
template <typename T>
void launch_kaczmarz_sweep(T* u, const T* uc, i64 n, i64 ld, int B, i64 start, i64 stop,
                           double proj_diag, cudaStream_t s) {
  require(0 <= start && start <= stop && stop <= n, "kaczmarz_sweep: window outside [0, n]");
  i64 j0 = start / 2, j1 = stop / 2;
  if (j1 <= j0) return;
  KzCoef<T> kz;
  int e;
  kz.proj_diag = (T)proj_diag;
  kz.pow2 = std::frexp(proj_diag, &e) == 0.5;
  kz.recip = (T)(kz.pow2 ? std::ldexp(1.0, 1 - e) : 1.0 / proj_diag);
  k_kaczmarz<T><<<grid_for(j1 - j0, B), dim3(TX, TY), 0, s>>>(u, uc, j0, j1, ld, B, kz);
  check_launch("kaczmarz_sweep");
}
template <typename T>
void launch_fourier_rhs(const double* coef, int K, i64 n, i64 ld, int B, T* f, T* uex,
                        cudaStream_t s) {
  k_fourier_rhs<T><<<grid_for(n, B), dim3(TX, TY), 0, s>>>(coef, K, n, ld, B, f, uex);
  check_launch("fourier_rhs");
}
template <typename T>
void launch_nonlinear_rhs(const double* scale, i64 n, i64 ld, int B, T* f, T* uex, cudaStream_t s) {
  k_nonlinear_rhs<T><<<grid_for(n, B), dim3(TX, TY), 0, s>>>(scale, n, ld, B, f, uex);
  check_launch("nonlinear_rhs");
}

// Self-test of the split division of the nonlinear smoother (div_by):
// q[i] = div_by(x[i], J[i], RN(1/J[i])) and the count of results that differ
// bitwise from the IEEE division x/J.
template <typename T>
__global__ void k_div_check(const T* __restrict__ x, const T* __restrict__ J, T* __restrict__ q,
                            i64 n, unsigned long long* bad) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const T a = x[i], b = J[i];
    const T v = div_by(a, b, xrcp(b)), w = xdiv(a, b);
    if (q) q[i] = v;
    bool same = sizeof(T) == 8 ? __double_as_longlong((double)v) == __double_as_longlong((double)w)
                               : __float_as_int((float)v) == __float_as_int((float)w);
    if (!same && !(v != v && w != w)) atomicAdd(bad, 1ull);
  }
}

template <typename T>
void launch_div_check(const T* x, const T* J, T* q, i64 n, unsigned long long* bad, cudaStream_t s) {
  require(n >= 0 && x && J && bad, "div_check: bad arguments");
  if (n == 0) return;
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_div_check<T><<<(unsigned)blocks, 256, 0, s>>>(x, J, q, n, bad);
  check_launch("div_check");
}

#define FMGSR_INST(T)                                                                          \
  template void launch_apply_operator<T>(const T*, T*, i64, i64, int, cudaStream_t);          \
  template void launch_restrict<T>(const T*, T*, i64, i64, int, cudaStream_t);                \
  template void launch_prolong_correction<T>(const T*, T*, i64, i64, int, cudaStream_t);      \
  template void launch_prolong_fmg<T>(const T*, T*, i64, i64, int, cudaStream_t);             \
  template void launch_restrict_tau<T>(const T*, const T*, T*, T*, i64, i64, int, int,        \
                                       cudaStream_t, bool);                                    \
  template void launch_direct_solve_nl<T>(const T*, T*, i64, i64, int, cudaStream_t);          \
  template void launch_fas_correct<T>(const T*, const T*, T*, i64, i64, int, cudaStream_t);   \
  template void launch_direct_solve<T>(const T*, T*, i64, i64, int, cudaStream_t, T*);            \
  template void launch_banded_lu_solve<T>(const T*, T*, i64, i64, int, T*, int*, cudaStream_t);  \
  template void launch_gs_sweep<T>(T*, const T*, i64, i64, int, double, i64, i64, bool,       \
                                   double, cudaStream_t);                                      \
  template void launch_kaczmarz_sweep<T>(T*, const T*, i64, i64, int, i64, i64, double,       \
                                         cudaStream_t);                                        \
  template void launch_fourier_rhs<T>(const double*, int, i64, i64, int, T*, T*, cudaStream_t); \
  template void launch_nonlinear_rhs<T>(const double*, i64, i64, int, T*, T*, cudaStream_t);    \
  template void launch_div_check<T>(const T*, const T*, T*, i64, unsigned long long*, cudaStream_t);
FMGSR_INST(double)
FMGSR_INST(float)
#undef FMGSR_INST

}  // namespace fmgsr
