// fmgsr_device.cuh -- device building blocks of the FMG-FAS-SR hot path.
//
// Layout: every level field is a row-major [n][ld] array, cell index i major,
// right-hand side r fastest (ld >= B).  One warp = one patch x 32 consecutive
// RHS columns, one lane = one (patch, rhs) Gauss-Seidel chain, so every load
// and store of a chain step is a coalesced 256 B (fp64) warp access.
//
// Arithmetic: every operation goes through the *_rn intrinsics below, so
// nvcc can never contract a multiply-add into an FMA.  Together with the
// reference's expression order this makes the CUDA path bit-identical to
// the reference numba lane (numba compiles without fastmath, no contraction;
// reference _kernels_numba.py:3-4).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fmgsr_internal.h"

namespace fmgsr {

typedef int64_t i64;

__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float xdiv(float a, float b) { return __fdiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// Two RHS columns per lane: V2<S> holds columns (2r, 2r+1) of a row, so a
// warp covers 64 adjacent columns and every staged row is one 16-byte (fp64)
// or 8-byte (fp32) access per lane.  Arithmetic is per component with the
// same *_rn intrinsics, so each column's result is bit-identical to the
// scalar chain; the lane simply runs two independent chains interleaved.
template <typename S>
struct alignas(2 * sizeof(S)) V2 {
  S x, y;
  V2() = default;
  __host__ __device__ constexpr explicit V2(double v) : x((S)v), y((S)v) {}
  __host__ __device__ constexpr V2(S a, S b) : x(a), y(b) {}
};
template <typename S>
__host__ __device__ inline bool operator==(const V2<S>& a, const V2<S>& b) {
  return a.x == b.x && a.y == b.y;
}
template <typename S>
__device__ __forceinline__ V2<S> xadd(V2<S> a, V2<S> b) { return V2<S>(xadd(a.x, b.x), xadd(a.y, b.y)); }
template <typename S>
__device__ __forceinline__ V2<S> xsub(V2<S> a, V2<S> b) { return V2<S>(xsub(a.x, b.x), xsub(a.y, b.y)); }
template <typename S>
__device__ __forceinline__ V2<S> xmul(V2<S> a, V2<S> b) { return V2<S>(xmul(a.x, b.x), xmul(a.y, b.y)); }
template <typename S>
__device__ __forceinline__ V2<S> xdiv(V2<S> a, V2<S> b) { return V2<S>(xdiv(a.x, b.x), xdiv(a.y, b.y)); }
// L2-coherent load (edge records written by another warp of the same launch)
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ V2<double> ldcg(const V2<double>* p) {
  double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return V2<double>(v.x, v.y);
}
__device__ __forceinline__ V2<float> ldcg(const V2<float>* p) {
  float2 v = __ldcg(reinterpret_cast<const float2*>(p));
  return V2<float>(v.x, v.y);
}
template <typename T>
struct LaneCols {  // RHS columns carried by one lane
  static constexpr int value = 1;
};
template <typename S>
struct LaneCols<V2<S>> {
  static constexpr int value = 2;
};

// Storage <-> arithmetic conversions.  Fields may be stored narrower than the
// arithmetic type (fp32 storage, fp64 arithmetic: values widen exactly on
// load and round to nearest once on store).
template <typename To>
__device__ __forceinline__ To cvt(double x);
template <typename To>
__device__ __forceinline__ To cvt(float x);
template <>
__device__ __forceinline__ double cvt<double>(double x) { return x; }
template <>
__device__ __forceinline__ float cvt<float>(float x) { return x; }
template <>
__device__ __forceinline__ double cvt<double>(float x) { return (double)x; }
template <>
__device__ __forceinline__ float cvt<float>(double x) { return __double2float_rn(x); }
template <typename To, typename S>
__device__ __forceinline__ To cvt(V2<S> x) {
  using E = decltype(To::x);
  return To(cvt<E>(x.x), cvt<E>(x.y));
}

// ---------------------------------------------------------------------------
// Gauss-Seidel cell updates, reference _kernels_numba.py:26-35.
//   interior : resid = f - inv_h2*((2u - uL) - uR), u += (omega*resid)/(2 inv_h2)
//   i == 0   : resid = f - inv_h2*(3u - uR),        u += (omega*resid)/(3 inv_h2)
//   i == n-1 : resid = f - inv_h2*(3u - uL),        u += (omega*resid)/(3 inv_h2)
// The interior divisor 2*4^k is a power of two, so the division is performed
// as an exact multiply by rdiag = 2^-(2k+1): both are the correctly rounded
// value of the same real number, hence bit-identical.  The boundary divisor
// 3*4^k is not a power of two and stays a true IEEE division.
// ---------------------------------------------------------------------------
template <typename T>
struct GsCoef {
  T inv_h2;  // 4^k
  T rdiag;   // 1 / (2 * 4^k), exact
  T diag_b;  // 3 * 4^k
  T omega;
  T diag_i;  // 2 * 4^k, exact (interior diagonal)
};

template <typename T>
__device__ __forceinline__ T gs_int(const GsCoef<T>& c, T uL, T u, T uR, T f) {
  T s = xsub(xsub(xmul(T(2), u), uL), uR);
  T resid = xsub(f, xmul(c.inv_h2, s));
  return xadd(u, xmul(xmul(c.omega, resid), c.rdiag));
}

template <typename T>
__device__ __forceinline__ T gs_bnd(const GsCoef<T>& c, T u, T nb, T f) {
  T s = xsub(xmul(T(3), u), nb);
  T resid = xsub(f, xmul(c.inv_h2, s));
  return xadd(u, xdiv(xmul(c.omega, resid), c.diag_b));
}

// One GS update of cell i in a level of n cells (domain rows first, as the
// reference tests i == 0 before i == n-1).
template <typename T>
__device__ __forceinline__ T gs_cell(const GsCoef<T>& c, i64 i, i64 n, T uL, T u, T uR,
                                     T f) {
  if (i == 0) return gs_bnd(c, u, uR, f);
  if (i == n - 1) return gs_bnd(c, u, uL, f);
  return gs_int(c, uL, u, uR, f);
}

// Nonlinear (-u'' + u^3 = f) Gauss-Seidel: one pointwise Newton step,
// r = f - (inv_h2*s + (u*u)*u), J = diag + 3(u*u), u += (omega*r)/J
// (oracle/fmgsr_oracle.c orc_gs_sweep_nl; the reference is linear only).
template <typename T>
__device__ __forceinline__ T gs_cell_nl(const GsCoef<T>& c, i64 i, i64 n, T uL, T u, T uR, T f) {
  T s, diag;
  if (i == 0) {
    s = xsub(xmul(T(3), u), uR);
    diag = c.diag_b;
  } else if (i == n - 1) {
    s = xsub(xmul(T(3), u), uL);
    diag = c.diag_b;
  } else {
    s = xsub(xsub(xmul(T(2), u), uL), uR);
    diag = xmul(T(2), c.inv_h2);
  }
  T uu = xmul(u, u);
  T r = xsub(f, xadd(xmul(c.inv_h2, s), xmul(uu, u)));
  T J = xadd(diag, xmul(T(3), uu));
  return xadd(u, xdiv(xmul(c.omega, r), J));
}

// x / J with y = RN(1/J) computed off the dependency chain.  q0 = RN(x y) is
// within 1.5 ulp of x/J; one Markstein correction q1 = RN(q0 + (x - J q0) y)
// makes it faithful, and by Markstein's theorem (y correctly rounded, q
// faithful, no underflow) the second correction yields RN(x/J), i.e. the
// __ddiv_rn result.  Outside the range where the theorem's no-underflow /
// no-overflow conditions hold (and for zeros, NaN, Inf) it falls back to the
// IEEE division.  tests/test_gpu_nonlinear.py checks it against xdiv.
__device__ __forceinline__ double xrcp(double J) { return __drcp_rn(J); }
__device__ __forceinline__ float xrcp(float J) { return __frcp_rn(J); }
__device__ __forceinline__ double xfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float xfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ bool div_safe(double x, double J) {
  const int ex = (__double2hiint(x) >> 20) & 0x7ff, eJ = (__double2hiint(J) >> 20) & 0x7ff;
  return (unsigned)(ex - (1023 - 800)) <= 1600u && (unsigned)(eJ - (1023 - 100)) <= 300u;
}
__device__ __forceinline__ bool div_safe(float x, float J) {
  const int ex = (__float_as_int(x) >> 23) & 0xff, eJ = (__float_as_int(J) >> 23) & 0xff;
  return (unsigned)(ex - (127 - 40)) <= 80u && (unsigned)(eJ - (127 - 20)) <= 90u;
}
// out of line so the compiler cannot if-convert the rare fallback into the
// fast path (it would evaluate both divisions)
template <typename T>
__device__ __noinline__ T div_slow(T x, T J) {
  return xdiv(x, J);
}
template <typename T>
__device__ __forceinline__ T div_by(T x, T J, T y) {
  T q = xmul(x, y);
  T r = xfma(-J, q, x);
  q = xfma(r, y, q);
  r = xfma(-J, q, x);
  q = xfma(r, y, q);
  if (!div_safe(x, J)) q = div_slow(x, J);
  return q;
}

// two-column lanes: the split division per component
template <typename S>
__device__ __forceinline__ V2<S> xrcp(V2<S> J) { return V2<S>(xrcp(J.x), xrcp(J.y)); }
template <typename S>
__device__ __forceinline__ V2<S> div_by(V2<S> x, V2<S> J, V2<S> y) {
  return V2<S>(div_by(x.x, J.x, y.x), div_by(x.y, J.y, y.y));
}

// Interior nonlinear GS cell (gs_cell_nl, i not a domain row) with the
// division split: J and 1/J depend only on the old u, so they are computed
// ahead of the uL dependency.
template <typename T, bool OMEGA1>
__device__ __forceinline__ T gs_int_nl(const GsCoef<T>& c, T uL, T u, T uR, T f) {
  T uu = xmul(u, u);
  T J = xadd(c.diag_i, xmul(T(3), uu));
  T y = xrcp(J);
  T s = xsub(xsub(xmul(T(2), u), uL), uR);
  T r = xsub(f, xadd(xmul(c.inv_h2, s), xmul(uu, u)));
  T x = OMEGA1 ? r : xmul(c.omega, r);
  return xadd(u, div_by(x, J, y));
}

template <typename T, bool OMEGA1>
__device__ __forceinline__ T gs_int_o(const GsCoef<T>& c, T uL, T u, T uR, T f) {
  T s = xsub(xsub(xmul(T(2), u), uL), uR);
  T resid = xsub(f, xmul(c.inv_h2, s));
  return xadd(u, xmul(OMEGA1 ? resid : xmul(c.omega, resid), c.rdiag));
}

// Kaczmarz projection of one pair onto its coarse value, reference
// _kernels_numba.py:53-56: r = uc - 0.5(a+b); t = r/proj_diag; a,b += 0.5 t.
// When proj_diag is a power of two (the reference's 0.5) the division is an
// exact multiply by its reciprocal.
// KP2: proj_diag is known to be a power of two (no division code at all)
template <bool KP2, typename T>
__device__ __forceinline__ void kaczmarz_pair_k(T& a, T& b, T uc, const KzCoef<T>& k) {
  T r = xsub(uc, xmul(T(0.5), xadd(a, b)));
  T t = KP2 ? xmul(r, k.recip) : xdiv(r, k.proj_diag);
  T h = xmul(T(0.5), t);
  a = xadd(a, h);
  b = xadd(b, h);
}
template <typename T>
__device__ __forceinline__ void kaczmarz_pair(T& a, T& b, T uc, const KzCoef<T>& k) {
  T r = xsub(uc, xmul(T(0.5), xadd(a, b)));
  T t = k.pow2 ? xmul(r, k.recip) : xdiv(r, k.proj_diag);
  T h = xmul(T(0.5), t);
  a = xadd(a, h);
  b = xadd(b, h);
}

// cp.async (LDGSTS) staging: each lane copies exactly the elements it will
// consume into its own shared-memory column, so a lane only ever waits on
// its own async groups (no warp or block synchronisation in the pipeline).
template <typename T>
__device__ __forceinline__ void cp_async(T* smem, const T* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(sizeof(T))
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// 1D bulk copies (TMA engine, cp.async.bulk) completing on an mbarrier: one
// lane moves a whole 32-column row segment per instruction.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// ---------------------------------------------------------------------------
// Pair sources: produce the smoother input u_in at fine cells (2q, 2q+1)
// together with f there, streaming in increasing q.
//   SRC_LOAD : u_in = u                                   (plain load)
//   SRC_CORR : u_in = u + P(uH - R u)   reference cycles.py:120-121,
//              stencils.py:39-64 (restrict, prolong_correction)
//   SRC_FMG  : u_in = Pi(uH)            reference stencils.py:67-105
// With CR the pair is projected (Kaczmarz) when it lies in the patch's pair
// range [ws//2, we//2): exactly the pairs the reference kaczmarz_sweep visits
// before the GS pass (_kernels_numba.py:42-57, 87-89), applied just in time.
// The raw rows of a pair are staged by cp.async into a per-lane ring slot
// (issue*), read back with fetch(), and turned into values by make*():
// make() handles every boundary row, make_fast() the interior only.
// ---------------------------------------------------------------------------
enum { SRC_LOAD = 0, SRC_CORR = 1, SRC_FMG = 2 };

template <typename T>
struct Raw {
  T a0, a1, h, g, f0, f1;
};

template <int SRC, bool CR>
struct SrcRows {
  // staged rows per pair: f(2) + LOAD u(2) | CORR u(2)+uH(1) | FMG uH(1), + uc(1) with CR
  static constexpr int R =
      2 + (SRC == SRC_LOAD ? 2 : SRC == SRC_CORR ? 3 : 1) + ((CR && SRC != SRC_FMG) ? 1 : 0);
};

template <typename T, int SRC, bool CR, typename M = T>
struct PairSource {
  static constexpr int R = SrcRows<SRC, CR>::R;
  // fields are stored as M (= T, or fp32 under fp64 arithmetic); the ring
  // stages them unconverted, fetch()/load()/init() widen to T
  const M* u;   // fine field, column-offset (LOAD, CORR)
  const M* uH;  // coarse field (CORR, FMG; CR target for FMG)
  const M* uc;  // CR target for LOAD / CORR
  const M* f;   // level right-hand side
  i64 ld, nc;   // row stride, number of pairs (= coarse cells)
  KzCoef<T> kz;
  i64 wlo, whi;  // Kaczmarz pair range
  i64 qlo, qhi;  // pairs that exist in memory (the whole level, or a shard's slab + halo)
  T s0, s1, s2, s3;
  // fast-issue row pointers (pair g): f row 2g, u row (LOAD 2g | CORR 2g+2),
  // uH row (CORR g+1 | FMG g+2), uc row g
  const M *pf, *pu, *ph, *pc;

  __device__ __forceinline__ i64 cl(i64 q) const { return q < qlo ? qlo : (q > qhi ? qhi : q); }

  // slot layout: sl[k * NT] for k < R (NT = threads per block)
  template <int NT>
  __device__ __forceinline__ void issue(M* sl, i64 g) const {
    i64 gg = cl(g);
    cp_async(sl, f + (2 * gg) * ld);
    cp_async(sl + NT, f + (2 * gg + 1) * ld);
    if (SRC == SRC_LOAD) {
      cp_async(sl + 2 * NT, u + (2 * gg) * ld);
      cp_async(sl + 3 * NT, u + (2 * gg + 1) * ld);
    } else if (SRC == SRC_CORR) {
      i64 g1 = cl(g + 1);
      cp_async(sl + 2 * NT, u + (2 * g1) * ld);
      cp_async(sl + 3 * NT, u + (2 * g1 + 1) * ld);
      cp_async(sl + 4 * NT, uH + g1 * ld);
    } else {
      cp_async(sl + 2 * NT, uH + cl(g + 2) * ld);
    }
    if (CR && SRC != SRC_FMG) cp_async(sl + (R - 1) * NT, uc + gg * ld);
  }

  // the R source rows of pair g (clamped), per-lane pointers shifted by -off
  // (off = lane gives the warp's 32-column row segment for a bulk copy)
  __device__ __forceinline__ void rows(i64 g, int off, const M* (&p)[R]) const {
    i64 gg = cl(g);
    p[0] = f + (2 * gg) * ld - off;
    p[1] = f + (2 * gg + 1) * ld - off;
    if (SRC == SRC_LOAD) {
      p[2] = u + (2 * gg) * ld - off;
      p[3] = u + (2 * gg + 1) * ld - off;
    } else if (SRC == SRC_CORR) {
      i64 g1 = cl(g + 1);
      p[2] = u + (2 * g1) * ld - off;
      p[3] = u + (2 * g1 + 1) * ld - off;
      p[4] = uH + g1 * ld - off;
    } else {
      p[2] = uH + cl(g + 2) * ld - off;
    }
    if (CR && SRC != SRC_FMG) p[R - 1] = uc + gg * ld - off;
  }

  __device__ __forceinline__ void fast_ptrs(i64 g) {
    pf = f + (2 * g) * ld;
    if (SRC == SRC_LOAD) pu = u + (2 * g) * ld;
    if (SRC == SRC_CORR) {
      pu = u + (2 * g + 2) * ld;
      ph = uH + (g + 1) * ld;
    }
    if (SRC == SRC_FMG) ph = uH + (g + 2) * ld;
    if (CR && SRC != SRC_FMG) pc = uc + g * ld;
  }

  // unclamped issue of the pair at the fast pointers, then advance one pair
  template <int NT>
  __device__ __forceinline__ void issue_fast(M* sl) {
    cp_async(sl, pf);
    cp_async(sl + NT, pf + ld);
    pf += 2 * ld;
    if (SRC == SRC_LOAD) {
      cp_async(sl + 2 * NT, pu);
      cp_async(sl + 3 * NT, pu + ld);
      pu += 2 * ld;
    } else if (SRC == SRC_CORR) {
      cp_async(sl + 2 * NT, pu);
      cp_async(sl + 3 * NT, pu + ld);
      cp_async(sl + 4 * NT, ph);
      pu += 2 * ld;
      ph += ld;
    } else {
      cp_async(sl + 2 * NT, ph);
      ph += ld;
    }
    if (CR && SRC != SRC_FMG) {
      cp_async(sl + (R - 1) * NT, pc);
      pc += ld;
    }
  }

  template <int NT>
  __device__ __forceinline__ Raw<T> fetch(const M* sl) const {
    Raw<T> r;
    r.f0 = cvt<T>(sl[0]);
    r.f1 = cvt<T>(sl[NT]);
    r.a0 = r.a1 = r.h = r.g = T(0);
    if (SRC == SRC_LOAD) {
      r.a0 = cvt<T>(sl[2 * NT]);
      r.a1 = cvt<T>(sl[3 * NT]);
    } else if (SRC == SRC_CORR) {
      r.a0 = cvt<T>(sl[2 * NT]);
      r.a1 = cvt<T>(sl[3 * NT]);
      r.h = cvt<T>(sl[4 * NT]);
    } else {
      r.h = cvt<T>(sl[2 * NT]);
    }
    if (CR && SRC != SRC_FMG) r.g = cvt<T>(sl[(R - 1) * NT]);
    return r;
  }

  // direct (uncached-path) load of a pair, for the chain head
  __device__ __forceinline__ Raw<T> load(i64 q) const {
    Raw<T> r;
    i64 qq = cl(q);
    r.f0 = cvt<T>(f[(2 * qq) * ld]);
    r.f1 = cvt<T>(f[(2 * qq + 1) * ld]);
    r.a0 = r.a1 = r.h = r.g = T(0);
    if (SRC == SRC_LOAD) {
      r.a0 = cvt<T>(u[(2 * qq) * ld]);
      r.a1 = cvt<T>(u[(2 * qq + 1) * ld]);
    } else if (SRC == SRC_CORR) {
      i64 q1 = cl(q + 1);
      r.a0 = cvt<T>(u[(2 * q1) * ld]);
      r.a1 = cvt<T>(u[(2 * q1 + 1) * ld]);
      r.h = cvt<T>(uH[q1 * ld]);
    } else {
      r.h = cvt<T>(uH[cl(q + 2) * ld]);
    }
    if (CR && SRC != SRC_FMG) r.g = cvt<T>(uc[qq * ld]);
    return r;
  }

  // sliding-window state before make(q), in two halves so that a chain head
  // can issue these loads before it stages its ring (the cp.async asm is a
  // compiler memory barrier: loads written after it are issued after it)
  T h0, h1, h2, h3, h4, h5;  // raw head values (init_loads -> init_finish)
  __device__ __forceinline__ void init_loads(i64 q) {
    if (SRC == SRC_CORR) {
      h2 = cvt<T>(u[(2 * q) * ld]);
      h3 = cvt<T>(u[(2 * q + 1) * ld]);
      h1 = cvt<T>(uH[q * ld]);
      if (q >= 1) {
        h4 = cvt<T>(u[(2 * q - 2) * ld]);
        h5 = cvt<T>(u[(2 * q - 1) * ld]);
        h0 = cvt<T>(uH[(q - 1) * ld]);
      }
    } else if (SRC == SRC_FMG) {
      h0 = cvt<T>(uH[cl(q - 2) * ld]);
      h1 = cvt<T>(uH[cl(q - 1) * ld]);
      h2 = cvt<T>(uH[cl(q) * ld]);
      h3 = cvt<T>(uH[cl(q + 1) * ld]);
    }
  }
  __device__ __forceinline__ void init_finish(i64 q) {
    if (SRC == SRC_CORR) {
      // s0 = c_{q-1}, s1 = c_q, s2 = u[2q], s3 = u[2q+1]; c_j = uH[j] - 0.5(u[2j] + u[2j+1])
      s2 = h2;
      s3 = h3;
      s1 = xsub(h1, xmul(T(0.5), xadd(s2, s3)));
      s0 = q >= 1 ? xsub(h0, xmul(T(0.5), xadd(h4, h5))) : T(0);
    } else if (SRC == SRC_FMG) {
      // s0..s3 = c[q-2], c[q-1], c[q], c[q+1] (clamped; boundary rows ignore them)
      s0 = h0;
      s1 = h1;
      s2 = h2;
      s3 = h3;
    }
  }
  __device__ __forceinline__ void init(i64 q) {
    init_loads(q);
    init_finish(q);
  }

  // interior FMG rows (stencils.py:90-97), then /128 as an exact scaling
  __device__ __forceinline__ void fmg_interior(T c4, T& e, T& o) const {
    e = xsub(xadd(xadd(xmul(T(-5), s0), xmul(T(35), s1)), xmul(T(105), s2)), xmul(T(7), s3));
    o = xsub(xadd(xadd(xmul(T(-7), s1), xmul(T(105), s2)), xmul(T(35), s3)), xmul(T(5), c4));
  }

  __device__ __forceinline__ void make(i64 q, const Raw<T>& r, T& v0, T& v1) {
    T target = r.g;
    if (SRC == SRC_LOAD) {
      v0 = r.a0;
      v1 = r.a1;
    } else if (SRC == SRC_CORR) {
      T c1 = xsub(r.h, xmul(T(0.5), xadd(r.a0, r.a1)));  // c_{q+1}
      T p0 = (q == 0) ? xmul(T(0.5), s1) : xmul(T(0.25), xadd(s0, xmul(T(3), s1)));
      T p1 = (q == nc - 1) ? xmul(T(0.5), s1) : xmul(T(0.25), xadd(xmul(T(3), s1), c1));
      v0 = xadd(s2, p0);
      v1 = xadd(s3, p1);
      s0 = s1;
      s1 = c1;
      s2 = r.a0;
      s3 = r.a1;
    } else {
      // prolong_fmg rows, reference stencils.py:85-104 (left-to-right sums, then /128)
      const T c0 = s0, c1 = s1, c2 = s2, c3 = s3, c4 = r.h;  // c[q-2 .. q+2]
      T e, o;
      if (q >= 2 && q <= nc - 3) {
        fmg_interior(c4, e, o);
      } else if (q == 0) {  // rows 0, 1 over c[0..2] = c2, c3, c4
        e = xsub(xmul(T(70), c2), xmul(T(2), c3));
        o = xsub(xadd(xmul(T(112), c2), xmul(T(35), c3)), xmul(T(5), c4));
      } else if (q == 1) {  // rows 2, 3 over c[0..3] = c1..c4
        e = xsub(xadd(xmul(T(40), c1), xmul(T(105), c2)), xmul(T(7), c3));
        o = xsub(xadd(xadd(xmul(T(-7), c1), xmul(T(105), c2)), xmul(T(35), c3)), xmul(T(5), c4));
      } else if (q == nc - 2) {  // rows nf-4, nf-3; c[n-1]=c3, c[n-2]=c2, c[n-3]=c1, c[n-4]=c0
        e = xsub(xadd(xadd(xmul(T(-7), c3), xmul(T(105), c2)), xmul(T(35), c1)), xmul(T(5), c0));
        o = xsub(xadd(xmul(T(40), c3), xmul(T(105), c2)), xmul(T(7), c1));
      } else {  // q == nc-1: rows nf-2, nf-1; c[n-1]=c2, c[n-2]=c1, c[n-3]=c0
        e = xsub(xadd(xmul(T(112), c2), xmul(T(35), c1)), xmul(T(5), c0));
        o = xsub(xmul(T(70), c2), xmul(T(2), c1));
      }
      v0 = xmul(e, T(0.0078125));  // x/128 == x*2^-7 exactly
      v1 = xmul(o, T(0.0078125));
      target = c2;
      s0 = c1;
      s1 = c2;
      s2 = c3;
      s3 = c4;
    }
    if (CR && q >= wlo && q < whi) kaczmarz_pair(v0, v1, target, kz);
  }

  // interior-only make (no boundary rows; CR pair always inside the window);
  // KP2: the Kaczmarz divisor is a power of two (the fast loops are unswitched
  // on it, so their bodies stay branch-free)
  template <bool KP2 = false>
  __device__ __forceinline__ void make_fast(const Raw<T>& r, T& v0, T& v1) {
    T target = r.g;
    if (SRC == SRC_LOAD) {
      v0 = r.a0;
      v1 = r.a1;
    } else if (SRC == SRC_CORR) {
      T c1 = xsub(r.h, xmul(T(0.5), xadd(r.a0, r.a1)));
      v0 = xadd(s2, xmul(T(0.25), xadd(s0, xmul(T(3), s1))));
      v1 = xadd(s3, xmul(T(0.25), xadd(xmul(T(3), s1), c1)));
      s0 = s1;
      s1 = c1;
      s2 = r.a0;
      s3 = r.a1;
    } else {
      T e, o;
      fmg_interior(r.h, e, o);
      v0 = xmul(e, T(0.0078125));
      v1 = xmul(o, T(0.0078125));
      target = s2;
      s0 = s1;
      s1 = s2;
      s2 = s3;
      s3 = r.h;
    }
    if (CR) {
      if (KP2) kaczmarz_pair_k<true>(v0, v1, target, kz);
      else kaczmarz_pair(v0, v1, target, kz);
    }
  }
};

// ---------------------------------------------------------------------------
// Restriction + tau epilogue, fused into the patch chain (reference
// stencils.py:108-125 coarse_rhs = R f + (L_H R u - R L u), cycles.py:101-102).
// The chain pushes its smoothed owned pairs in order; coarse cell j-1 is
// emitted one pair late (it needs R u at j).  The patch's first and last
// coarse cells need two smoothed fine cells of the neighbouring patch: they
// are completed by whichever of the two neighbour warps finishes second
// (edge records + a parity counter, see edge_arrive).  Requires W >= 4.
// ---------------------------------------------------------------------------
template <typename T>
struct EdgeRec {
  T v[5];
};

template <typename T, typename M = T>
struct Epilogue {
  T inv_h2, inv_H2;
  bool left_dom, right_dom, write_uH;
  M* uH_out;  // column-offset (fields stored as M)
  M* fH_out;  // column-offset
  i64 ld, nc;
  T up2, up1, Lprev, Rm2, Rm1, Rfm1;
  EdgeRec<T> left;  // u[os], u[os+1], Lu[os+1], Ru_{j0+1}, Rf_{j0}
  int cnt;

  __device__ __forceinline__ void push(i64 j, T a, T b, T f0, T f1, bool store) {
    T Rj = xmul(T(0.5), xadd(a, b));
    T Rfj = xmul(T(0.5), xadd(f0, f1));
    if (write_uH && store) uH_out[j * ld] = cvt<M>(Rj);
    if (cnt == 0) {
      if (left_dom) {
        Lprev = xmul(xsub(xmul(T(3), a), b), inv_h2);  // Lu[0]
      } else {
        left.v[0] = a;
        left.v[1] = b;
        left.v[4] = Rfj;
      }
    } else {
      T Lodd = xmul(xsub(xsub(xmul(T(2), up1), up2), a), inv_h2);  // Lu[2j-1]
      if (cnt == 1 && !left_dom) {
        left.v[2] = Lodd;  // Lu[os+1]
        left.v[3] = Rj;    // Ru_{j0+1}
      } else {
        T RL = xmul(T(0.5), xadd(Lprev, Lodd));
        T LH = (j - 1 == 0) ? xmul(xsub(xmul(T(3), Rm1), Rj), inv_H2)
                            : xmul(xsub(xsub(xmul(T(2), Rm1), Rm2), Rj), inv_H2);
        if (store) fH_out[(j - 1) * ld] = cvt<M>(xadd(Rfm1, xsub(LH, RL)));
      }
      Lprev = xmul(xsub(xsub(xmul(T(2), a), up1), b), inv_h2);  // Lu[2j]
    }
    up2 = a;
    up1 = b;
    Rm2 = Rm1;
    Rm1 = Rj;
    Rfm1 = Rfj;
    cnt++;
  }

  // steady-state push (cnt >= 2, coarse cell j-1 interior): pointer-walking
  // version of push() for the chain's fast loop; call fast_begin(j) first.
  M* puH;
  M* pfH;
  __device__ __forceinline__ void fast_begin(i64 j) {
    puH = uH_out ? uH_out + j * ld : nullptr;
    pfH = fH_out + (j - 1) * ld;
  }
  // WUH: store R u (uniform per launch); every lane stores (visit_kernel's rr)
  template <bool WUH>
  __device__ __forceinline__ void push_fast(T a, T b, T f0, T f1) {
    T Rj = xmul(T(0.5), xadd(a, b));
    T Rfj = xmul(T(0.5), xadd(f0, f1));
    if (WUH) {
      *puH = cvt<M>(Rj);
      puH += ld;
    }
    T Lodd = xmul(xsub(xsub(xmul(T(2), up1), up2), a), inv_h2);
    T RL = xmul(T(0.5), xadd(Lprev, Lodd));
    T LH = xmul(xsub(xsub(xmul(T(2), Rm1), Rm2), Rj), inv_H2);
    *pfH = cvt<M>(xadd(Rfm1, xsub(LH, RL)));
    pfH += ld;
    Lprev = xmul(xsub(xsub(xmul(T(2), a), up1), b), inv_h2);
    up2 = a;
    up1 = b;
    Rm2 = Rm1;
    Rm1 = Rj;
    Rfm1 = Rfj;
    cnt++;
  }

  // after the last owned pair: close the domain end or build the right record
  __device__ __forceinline__ void finish(bool store, EdgeRec<T>& right) {
    if (right_dom) {
      T Llast = xmul(xsub(xmul(T(3), up1), up2), inv_h2);  // Lu[n-1]
      T RL = xmul(T(0.5), xadd(Lprev, Llast));
      T LH = xmul(xsub(xmul(T(3), Rm1), Rm2), inv_H2);
      if (store) fH_out[(nc - 1) * ld] = cvt<M>(xadd(Rfm1, xsub(LH, RL)));
    } else {
      right.v[0] = up2;    // u[s-2]
      right.v[1] = up1;    // u[s-1]
      right.v[2] = Lprev;  // Lu[s-2]
      right.v[3] = Rm2;    // Ru_{jL-1}
      right.v[4] = Rfm1;   // Rf_{jL}
    }
  }
};

// Complete coarse cells s/2-1 and s/2 of the patch boundary at fine cell s
// from the left record (slots 0-4) and the right record (slots 5-9).
// NL: the records' L values are N u = L u + u^3 (nonlinear tau), and the two
// fine and two coarse operator values formed here get their cubes added in the
// k_restrict_tau order.
template <typename T>
__device__ __forceinline__ T cube(T x) {
  return xmul(xmul(x, x), x);
}
template <typename T, bool NL = false>
__device__ __forceinline__ void edge_finish(const T* L, const T* R, T inv_h2, T inv_H2, T& fL,
                                            T& fR) {
  const T um2 = L[0], um1 = L[1], Lm2 = L[2], RuLm1 = L[3], RfL = L[4];
  const T u0 = R[0], u1 = R[1], L1 = R[2], RuRp1 = R[3], RfR = R[4];
  T Lm1 = xmul(xsub(xsub(xmul(T(2), um1), um2), u0), inv_h2);
  T L0 = xmul(xsub(xsub(xmul(T(2), u0), um1), u1), inv_h2);
  if (NL) {
    Lm1 = xadd(Lm1, cube(um1));
    L0 = xadd(L0, cube(u0));
  }
  T RuL = xmul(T(0.5), xadd(um2, um1));
  T RuR = xmul(T(0.5), xadd(u0, u1));
  T RLL = xmul(T(0.5), xadd(Lm2, Lm1));
  T RLR = xmul(T(0.5), xadd(L0, L1));
  T LHL = xmul(xsub(xsub(xmul(T(2), RuL), RuLm1), RuR), inv_H2);
  T LHR = xmul(xsub(xsub(xmul(T(2), RuR), RuL), RuRp1), inv_H2);
  if (NL) {
    LHL = xadd(LHL, cube(RuL));
    LHR = xadd(LHR, cube(RuR));
  }
  fL = xadd(RfL, xsub(LHL, RLL));
  fR = xadd(RfR, xsub(LHR, RLR));
}

// Edge protocol for one boundary (index bi, boundary fine cell s).  Each of
// the two neighbour warps writes its 5-slot record, fences, and bumps the
// boundary's counter; the warp that sees an odd old value arrived second and
// finishes both coarse cells.  Every boundary receives exactly two arrivals
// per visit, so the parity test stays valid across visits without resets.
template <typename T, bool NL = false, typename M = T>
__device__ __forceinline__ void edge_arrive(T* E, int* cnt, i64 ldE, int nrg, i64 bi, int side,
                                            const EdgeRec<T>& rec, int lane, int rg, int r,
                                            bool store, M* fH, i64 ld, i64 s, T inv_h2,
                                            T inv_H2) {
  T* mine = E + (bi * 10 + side * 5) * ldE + r;
#pragma unroll
  for (int k = 0; k < 5; k++) mine[k * ldE] = rec.v[k];
  __threadfence();
  __syncwarp();
  int old = 0;
  if (lane == 0) old = atomicAdd(cnt + bi * nrg + rg, 1);
  old = __shfl_sync(0xffffffffu, old, 0);
  if (old & 1) {
    __threadfence();
    const T* base = E + bi * 10 * ldE + r;
    T Lr[5], Rr[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
      Lr[k] = ldcg(base + k * ldE);
      Rr[k] = ldcg(base + (5 + k) * ldE);
    }
    T fL, fR;
    edge_finish<T, NL>(Lr, Rr, inv_h2, inv_H2, fL, fR);
    if (store) {
      fH[(s / 2 - 1) * ld] = cvt<M>(fL);
      fH[(s / 2) * ld] = cvt<M>(fR);
    }
  }
}

// Both boundaries of a patch in one round: the two records are written, ONE
// fence, both counters bumped back to back by lane 0, then each boundary this
// warp reached second is completed -- the edge_arrive protocol with one memory
// round trip fewer per warp.  doL: the left boundary (index biL = p, this warp
// is its side 1, fine cell sL = os); doR: the right one (biR = p + 1, side 0,
// sR = oe).
template <typename T, bool NL = false, typename M = T>
__device__ __forceinline__ void edge_arrive2(T* E, int* cnt, i64 ldE, int nrg, int lane, int rg,
                                             int r, bool store, M* fH, i64 ld, T inv_h2,
                                             T inv_H2, bool doL, i64 biL,
                                             const EdgeRec<T>& recL, i64 sL, bool doR, i64 biR,
                                             const EdgeRec<T>& recR, i64 sR) {
  if (!doL && !doR) return;
  if (doL) {
    T* mine = E + (biL * 10 + 5) * ldE + r;
#pragma unroll
    for (int k = 0; k < 5; k++) mine[k * ldE] = recL.v[k];
  }
  if (doR) {
    T* mine = E + (biR * 10) * ldE + r;
#pragma unroll
    for (int k = 0; k < 5; k++) mine[k * ldE] = recR.v[k];
  }
  __threadfence();
  __syncwarp();
  int oL = 0, oR = 0;
  if (lane == 0) {
    if (doL) oL = atomicAdd(cnt + biL * nrg + rg, 1);
    if (doR) oR = atomicAdd(cnt + biR * nrg + rg, 1);
  }
  oL = __shfl_sync(0xffffffffu, oL, 0);
  oR = __shfl_sync(0xffffffffu, oR, 0);
  const bool finL = doL && (oL & 1), finR = doR && (oR & 1);
  if (!finL && !finR) return;
  __threadfence();
  auto finish = [&](i64 bi, i64 s) {
    const T* base = E + bi * 10 * ldE + r;
    T Lr[5], Rr[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
      Lr[k] = ldcg(base + k * ldE);
      Rr[k] = ldcg(base + (5 + k) * ldE);
    }
    T fL, fR;
    edge_finish<T, NL>(Lr, Rr, inv_h2, inv_H2, fL, fR);
    if (store) {
      fH[(s / 2 - 1) * ld] = cvt<M>(fL);
      fH[(s / 2) * ld] = cvt<M>(fR);
    }
  };
  if (finL) finish(biL, sL);
  if (finR) finish(biR, sR);
}

}  // namespace fmgsr
