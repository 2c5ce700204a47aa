// kernels_coarse.cu -- the coarse end of the hierarchy, resident on chip.
//
// Below a cutoff level Lc every level visit of the FMG cycle is a few
// microseconds of latency-bound work, so launching one grid per visit (the
// reference's horizontal order) would be dominated by launch and pipeline
// fill.  Right-hand sides are independent, so one CTA owns a group of CW RHS
// columns and runs *all* visits of levels m0..Lc for them out of shared
// memory, separated only by __syncthreads():
//   mode 0 (coarse FMG): the coarsest direct solve and FMG steps m0+1..Lc
//                        (reference cycles.py:178-199 for those levels);
//   mode 1 (V segment) : for a step t > Lc, the part of the V-cycle below
//                        Lc+1: down leg Lc..m0+1, direct solve, up leg
//                        m0+1..Lc (cycles.py:95-134).
// Operators are the exact-order device functions shared with the grid
// kernels, so results stay bit-identical to the reference.
//
// The same launch also hosts the multi-level restriction of the forcing
// (the f cascade, cycles.py:178-180).
#include <cmath>
#include <cstdio>
#include <type_traits>

#include "fmgsr_device.cuh"

#include "fmgsr_internal.h"

namespace fmgsr {

namespace {

constexpr int CNT = 512;  // threads per coarse CTA

// 2^e built from its exponent bits (exact; no int -> fp conversion)
__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
template <typename T>
__device__ __forceinline__ T pow4(int l) {
  return (T)pow2d(2 * l);
}

// Shared-memory layout of the coarse hierarchy for CW columns: level l keeps
// u0, u1, f (n_l x CW each, cell-major, column fastest) at offset
// 3 CW (2^l - 2^m0); a level's current u buffer is one bit of `curmask`.
// Everything is addressed arithmetically (no per-level tables), so nothing
// spills to local memory.
template <typename T, int CW, typename M = T>
struct CoarseCtx {
  const CoarseArgs<T, M>& a;
  T* sm;
  const T* dfac;  // direct-solve factor d[n0], e[n0], RN(1/d)[n0]
  const T* efac;
  const T* rfac;
  T* pjb = nullptr;  // projected copy of an SR level's smoother input (a.pj)
  T* fob = nullptr;  // on-chip f cascade (a.fo): level l at fob + CW (2^l - 2^m0)
  __device__ __forceinline__ T* FO(int l) const { return fob + CW * ((1 << l) - (1 << a.m0)); }
  // f cascade of cycles.py:178-180 in shared memory: the same pair averages,
  // level by level, as k_cascade
  __device__ void cascade_on_chip(int m) {
    load(FO(m), a.forig[m], 1 << m);
    bar("load", m);
    for (int l = m - 1; l >= a.m0; l--) {
      const T* src = FO(l + 1);
      T* dst = FO(l);
      for (int e = threadIdx.x; e < (1 << l) * CW; e += blockDim.x) {
        const int j = e / CW, c = e % CW;
        dst[e] = xmul(T(0.5), xadd(src[(2 * j) * CW + c], src[(2 * j + 1) * CW + c]));
      }
      bar("cascade", l);
    }
  }
  __device__ void copy(T* dst, const T* src, int n) {
    for (int e = threadIdx.x; e < n * CW; e += blockDim.x) dst[e] = src[e];
  }
  int c0;
  unsigned curmask;
  __device__ CoarseCtx(const CoarseArgs<T, M>& args) : a(args) {}

  __device__ __forceinline__ int nlev(int l) const { return 1 << l; }
  __device__ __forceinline__ T* U(int l, int w) const {
    return sm + 3 * CW * ((1 << l) - (1 << a.m0)) + w * CW * (1 << l);
  }
  __device__ __forceinline__ T* Fl(int l) const { return U(l, 2); }
  __device__ __forceinline__ int cur(int l) const { return (curmask >> l) & 1; }
  __device__ __forceinline__ void flip(int l) { curmask ^= 1u << l; }
  __device__ __forceinline__ void set0(int l) { curmask &= ~(1u << l); }

  __device__ bool sr(int l) const { return l > a.m - a.n_sr; }

  // barrier between phases; FMGSR_COARSE_TRACE=1 makes CTA 0 printf the
  // clock at every barrier (phase-latency profiling, off by default)
  int nbar;
  struct Trace {
    long long t[256];
    const char* what[256];
    int lvl[256];
  };
  __device__ __forceinline__ Trace* trace() const {
    __shared__ Trace tr;
    return &tr;
  }
  __device__ __forceinline__ void bar(const char* what, int l) {
    __syncthreads();
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && nbar < 256) {
      Trace* tr = trace();
      tr->t[nbar] = clock64();
      tr->what[nbar] = what;
      tr->lvl[nbar++] = l;
    }
  }
  __device__ void dump() {
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
      const Trace* tr = trace();
      for (int i = 1; i < nbar; i++)
        printf("coarse-trace %d %lld %s %d\n", i, tr->t[i] - tr->t[i - 1], tr->what[i], tr->lvl[i]);
    }
  }

  // global -> shared by cp.async: every element in flight at once, one wait
  // (narrower storage: plain loads, widened exactly)
  __device__ void load(T* dst, const M* src, int n) {
    for (int e = threadIdx.x; e < n * CW; e += blockDim.x) {
      int i = e / CW, c = e % CW, col = c0 + c;
      if (col < a.B) {
        if constexpr (std::is_same<T, M>::value) cp_async(dst + e, src + (i64)i * a.ld + col);
        else dst[e] = cvt<T>(src[(i64)i * a.ld + col]);
      } else {
        dst[e] = T(0);
      }
    }
    cp_commit();
    cp_wait<0>();
  }
  __device__ void store(M* dst, const T* src, int n) {
    for (int e = threadIdx.x; e < n * CW; e += blockDim.x) {
      int i = e / CW, c = e % CW, col = c0 + c;
      if (col < a.B) dst[(i64)i * a.ld + col] = cvt<M>(src[e]);
    }
  }

  // ---- on-the-fly operators on one column (pointer already column-offset) ----
  // prolong_fmg row i (stencils.py:67-105) from coarse column s of nc cells
  __device__ __forceinline__ T fmg_row(const T* s, int i, int nc) const {
    const int nf = 2 * nc;
#define C(k) s[(k) * CW]
    T v;
    if (i >= 4 && i < nf - 4) {
      if ((i & 1) == 0) {
        int q = i >> 1;
        v = xsub(xadd(xadd(xmul(T(-5), C(q - 2)), xmul(T(35), C(q - 1))), xmul(T(105), C(q))),
                 xmul(T(7), C(q + 1)));
      } else {
        int q = i >> 1;
        v = xsub(xadd(xadd(xmul(T(-7), C(q - 1)), xmul(T(105), C(q))), xmul(T(35), C(q + 1))),
                 xmul(T(5), C(q + 2)));
      }
    } else if (i == 0) v = xsub(xmul(T(70), C(0)), xmul(T(2), C(1)));
    else if (i == 1) v = xsub(xadd(xmul(T(112), C(0)), xmul(T(35), C(1))), xmul(T(5), C(2)));
    else if (i == 2) v = xsub(xadd(xmul(T(40), C(0)), xmul(T(105), C(1))), xmul(T(7), C(2)));
    else if (i == 3)
      v = xsub(xadd(xadd(xmul(T(-7), C(0)), xmul(T(105), C(1))), xmul(T(35), C(2))), xmul(T(5), C(3)));
    else if (i == nf - 4)
      v = xsub(xadd(xadd(xmul(T(-7), C(nc - 1)), xmul(T(105), C(nc - 2))), xmul(T(35), C(nc - 3))),
               xmul(T(5), C(nc - 4)));
    else if (i == nf - 3)
      v = xsub(xadd(xmul(T(40), C(nc - 1)), xmul(T(105), C(nc - 2))), xmul(T(7), C(nc - 3)));
    else if (i == nf - 2)
      v = xsub(xadd(xmul(T(112), C(nc - 1)), xmul(T(35), C(nc - 2))), xmul(T(5), C(nc - 3)));
    else v = xsub(xmul(T(70), C(nc - 1)), xmul(T(2), C(nc - 2)));
#undef C
    return xmul(v, T(0.0078125));
  }

  // u[i] + P(uH - R u)[i] (cycles.py:120-121, stencils.py:39-64); u has nf cells
  __device__ __forceinline__ T corr_row(const T* u, const T* uH, int i, int nf) const {
    const int nc = nf >> 1;
    auto cc = [&](int j) {
      return xsub(uH[j * CW], xmul(T(0.5), xadd(u[(2 * j) * CW], u[(2 * j + 1) * CW])));
    };
    T p;
    if (i == 0) p = xmul(T(0.5), cc(0));
    else if (i == nf - 1) p = xmul(T(0.5), cc(nc - 1));
    else if (i & 1) {
      int j = (i - 1) >> 1;
      p = xmul(T(0.25), xadd(xmul(T(3), cc(j)), cc(j + 1)));
    } else {
      int j = (i - 2) >> 1;
      p = xmul(T(0.25), xadd(cc(j), xmul(T(3), cc(j + 1))));
    }
    return xadd(u[i * CW], p);
  }

  // coarse_rhs at coarse cell j (stencils.py:108-125) from fine u, f of nf
  // cells on level lf (ih = 4^lf, iH = 4^(lf-1))
  __device__ __forceinline__ T crhs_row(const T* u, const T* f, int j, int nf, T ih, T iH) const {
    const int nc = nf >> 1;
    auto ru = [&](int k) { return xmul(T(0.5), xadd(u[(2 * k) * CW], u[(2 * k + 1) * CW])); };
    auto lu = [&](int i) {
      T s;
      if (i == 0) s = xsub(xmul(T(3), u[0]), u[CW]);
      else if (i == nf - 1) s = xsub(xmul(T(3), u[(nf - 1) * CW]), u[(nf - 2) * CW]);
      else s = xsub(xsub(xmul(T(2), u[i * CW]), u[(i - 1) * CW]), u[(i + 1) * CW]);
      return xmul(s, ih);
    };
    T Rj = ru(j);
    T LH;
    if (j == 0) LH = xmul(xsub(xmul(T(3), Rj), ru(1)), iH);
    else if (j == nc - 1) LH = xmul(xsub(xmul(T(3), Rj), ru(nc - 2)), iH);
    else LH = xmul(xsub(xsub(xmul(T(2), Rj), ru(j - 1)), ru(j + 1)), iH);
    T RL = xmul(T(0.5), xadd(lu(2 * j), lu(2 * j + 1)));
    T Rf = xmul(T(0.5), xadd(f[(2 * j) * CW], f[(2 * j + 1) * CW]));
    return xadd(Rf, xsub(LH, RL));
  }

  // ---- data-parallel stencil phases (one thread per output element) ---------------
  __device__ void phase_fmg(T* dst, const T* uH, int l) {  // dst = Pi uH (level l)
    const int nf = nlev(l);
    for (int e = threadIdx.x; e < nf * CW; e += blockDim.x)
      dst[e] = fmg_row(uH + e % CW, e / CW, nf >> 1);
  }
  __device__ void phase_corr(T* dst, const T* u, const T* uH, int l) {  // u + P(uH - R u)
    const int nf = nlev(l);
    for (int e = threadIdx.x; e < nf * CW; e += blockDim.x)
      dst[e] = corr_row(u + e % CW, uH + e % CW, e / CW, nf);
  }
  __device__ void phase_restrict(T* uH, T* fH, const T* u, const T* f, int l) {  // level l -> l-1
    const int nf = nlev(l), nc = nf >> 1;
    const T ih = pow4<T>(l), iH = pow4<T>(l - 1);
    for (int e = threadIdx.x; e < nc * CW; e += blockDim.x) {
      const int j = e / CW, c = e % CW;
      fH[e] = crhs_row(u + c, f + c, j, nf, ih, iH);
      uH[e] = xmul(T(0.5), xadd(u[(2 * j) * CW + c], u[(2 * j + 1) * CW + c]));
    }
  }

  // Kaczmarz projection of every pair of the level (the values the CR pass gives
  // the pairs a patch projects, _kernels_numba.py:42-57): pj = projected u_in
  __device__ void phase_project(T* pj, const T* uin, const T* uc, int l) {
    const int nc = nlev(l) >> 1;
    for (int e = threadIdx.x; e < nc * CW; e += blockDim.x) {
      const int j = e / CW, c = e % CW;
      T aa = uin[(2 * j) * CW + c], bb = uin[(2 * j + 1) * CW + c];
      kaczmarz_pair(aa, bb, uc[j * CW + c], a.kz);
      pj[(2 * j) * CW + c] = aa;
      pj[(2 * j + 1) * CW + c] = bb;
    }
  }

  // ---- patch chains: additive ns = 1 smoother (_kernels_numba.py:60-92) -----------
  // one chain per (patch, column) over the precomputed input uin; Kaczmarz (CR)
  // per pair inside the window; domain-boundary rows peeled off the loop.
  template <bool CR>
  __device__ void chains(int l, const T* uin, const T* f, const T* uc, T* out,
                         const T* pj = nullptr) {
    const int n = nlev(l), W = (int)a.W[l], b = (int)a.b[l];
    const int P = n / W;
    GsCoef<T> gc;
    gc.inv_h2 = pow4<T>(l);
    gc.rdiag = (T)pow2d(-(2 * l + 1));
    gc.diag_b = xmul(T(3), gc.inv_h2);
    gc.omega = (T)a.omega;
    gc.diag_i = xmul(T(2), gc.inv_h2);
    for (int k = threadIdx.x; k < P * CW; k += blockDim.x) {
      const int p = k / CW, c = k % CW;
      const int os = p * W, oe = os + W;
      const int ws = os - b > 0 ? os - b : 0;
      const int we = oe + b < n ? oe + b : n;
      const int wlo = ws >> 1, whi = we >> 1;
      const T* ui = uin + c;
      const T* fc = f + c;
      T* oc = out + c;
      const T* pc = pj ? pj + c : nullptr;
      auto val = [&](int x) -> T {
        if (!CR) return ui[x * CW];
        const int j = x >> 1;
        if (pc) return (j >= wlo && j < whi) ? pc[x * CW] : ui[x * CW];
        T v = ui[x * CW];
        if (j >= wlo && j < whi) {
          T aa = ui[(2 * j) * CW], bb = ui[(2 * j + 1) * CW];
          kaczmarz_pair(aa, bb, uc[j * CW + c], a.kz);
          v = (x & 1) ? bb : aa;
        }
        return v;
      };
      int i = ws;
      T uL = ws > 0 ? val(ws - 1) : T(0);
      T cu = val(ws);
      T nx = val(ws + 1);  // n >= 8 on every smoothed level
      if (i == 0) {
        T v = gs_bnd(gc, cu, nx, fc[0]);
        if (os == 0) oc[0] = v;
        uL = v;
        cu = nx;
        nx = val(2);
        i = 1;
      }
      const int iend = oe < n - 1 ? oe : n - 1;
      // f of the next cell is read one iteration ahead, so its shared-memory
      // latency overlaps the current cell's dependent fp64 chain
      T fi = fc[i * CW];
      for (; i < iend; i++) {
        T nn = val(i + 2 < n ? i + 2 : n - 1);
        const T fnext = fc[(i + 1) * CW];  // i + 1 <= n - 1
        T v = gs_int(gc, uL, cu, nx, fi);
        if (i >= os) oc[i * CW] = v;
        uL = v;
        cu = nx;
        nx = nn;
        fi = fnext;
      }
      if (oe == n) oc[(n - 1) * CW] = gs_bnd(gc, cu, uL, fc[(n - 1) * CW]);
    }
  }

  // LAPACK ?ptsv order (smoothers.py:210-225): dptts2 with the shared factor
  __device__ void direct(T* u) {
    const int n = nlev(a.m0);
    const T* f = Fl(a.m0);
    for (int c = threadIdx.x; c < CW; c += blockDim.x) {
      T prev = f[c];
      u[c] = prev;
      for (int i = 1; i < n; i++) {
        prev = xsub(f[i * CW + c], xmul(prev, efac[i - 1]));
        u[i * CW + c] = prev;
      }
      // x / d[i] as div_by with the reciprocals of the (constant) factor:
      // bitwise the IEEE quotient, and off the backward recurrence's chain
      T nx = div_by(prev, dfac[n - 1], rfac[n - 1]);
      u[(n - 1) * CW + c] = nx;
      for (int i = n - 2; i >= 0; i--) {
        nx = xsub(div_by(u[i * CW + c], dfac[i], rfac[i]), xmul(nx, efac[i]));
        u[i * CW + c] = nx;
      }
    }
  }

  // ---- level visits (each phase ends with a barrier) ----------------------------
  __device__ void visit_top(int t) {  // Pi, pre-smooth, restrict + tau
    const int h = cur(t - 1);
    phase_fmg(U(t, 1), U(t - 1, h), t);
    bar("T.fmg", t);
    chains<false>(t, U(t, 1), Fl(t), nullptr, U(t, 0));
    set0(t);
    bar("T.smooth", t);
    phase_restrict(U(t - 1, h ^ 1), Fl(t - 1), U(t, 0), Fl(t), t);
    flip(t - 1);
    bar("T.restrict", t);
  }
  __device__ void visit_down(int l) {
    const int c = cur(l);
    chains<false>(l, U(l, c), Fl(l), nullptr, U(l, c ^ 1));
    flip(l);
    bar("D.smooth", l);
    const int h = cur(l - 1);
    phase_restrict(U(l - 1, h ^ 1), Fl(l - 1), U(l, c ^ 1), Fl(l), l);
    flip(l - 1);
    bar("D.restrict", l);
  }
  __device__ void visit_direct() {
    const int c = cur(a.m0);
    direct(U(a.m0, c ^ 1));
    flip(a.m0);
    bar("direct", a.m0);
  }
  __device__ void visit_up(int l) {
    const int c = cur(l);
    const T* uH = U(l - 1, cur(l - 1));
    const bool s = sr(l);
    if (s) phase_fmg(U(l, c ^ 1), uH, l);
    else phase_corr(U(l, c ^ 1), U(l, c), uH, l);
    bar("U.prolong", l);
    if (s && pjb) {  // project every pair once instead of per cell inside the chains
      phase_project(pjb, U(l, c ^ 1), uH, l);
      bar("U.project", l);
    }
    if (s) chains<true>(l, U(l, c ^ 1), Fl(l), uH, U(l, c), pjb);
    else chains<false>(l, U(l, c ^ 1), Fl(l), nullptr, U(l, c));
    bar("U.smooth", l);
  }
};

template <typename T, int CW, typename M = T>
__global__ void __launch_bounds__(CNT, 1) coarse_kernel(const CoarseArgs<T, M> a) {
  extern __shared__ __align__(16) unsigned char coarse_smem[];
  CoarseCtx<T, CW, M> x(a);
  x.sm = reinterpret_cast<T*>(coarse_smem);
  x.c0 = blockIdx.x * CW;
  x.curmask = 0;
  x.nbar = 0;
  x.bar("start", 0);
  const int m0 = a.m0, Lc = a.Lc;
  const int n0 = 1 << m0;
  T* d = x.sm + 3 * CW * ((1 << (Lc + 1)) - (1 << m0));
  T* e = d + n0;
  if (threadIdx.x == 0) {  // dpttrf, as in k_direct_solve
    T ih = pow4<T>(m0);
    for (int i = 0; i < n0; i++) d[i] = xmul(T(2), ih);
    d[0] = xmul(T(3), ih);
    d[n0 - 1] = xmul(T(3), ih);
    for (int i = 0; i < n0 - 1; i++) e[i] = -ih;
    for (int i = 0; i < n0 - 1; i++) {
      T ei = e[i];
      e[i] = xdiv(ei, d[i]);
      d[i + 1] = xsub(d[i + 1], xmul(e[i], ei));
    }
    for (int i = 0; i < n0; i++) e[n0 + i] = xrcp(d[i]);
  }
  x.dfac = d;
  x.efac = e;
  x.rfac = e + n0;
  x.pjb = a.pj ? e + 2 * n0 : nullptr;
  x.fob = a.fo ? e + 2 * n0 + (a.pj ? (1 << Lc) * CW : 0) : nullptr;
  if (a.mode == 0) {
    if (x.fob) {
      x.cascade_on_chip(Lc);
      x.copy(x.Fl(m0), x.FO(m0), n0);
    } else {
      x.load(x.Fl(m0), a.forig[m0], n0);
    }
    x.bar("load", m0);
    x.visit_direct();
    for (int t = m0 + 1; t <= Lc; t++) {
      if (x.fob) x.copy(x.Fl(t), x.FO(t), 1 << t);
      else x.load(x.Fl(t), a.forig[t], 1 << t);
      x.bar("load", t);
      x.visit_top(t);
      for (int l = t - 1; l > m0; l--) x.visit_down(l);
      x.visit_direct();
      for (int l = m0 + 1; l <= t; l++) x.visit_up(l);
    }
  } else {
    x.load(x.U(Lc, 0), a.u_top, 1 << Lc);
    x.load(x.Fl(Lc), a.f_top, 1 << Lc);
    x.bar("load", Lc);
    for (int l = Lc; l > m0; l--) x.visit_down(l);
    x.visit_direct();
    for (int l = m0 + 1; l <= Lc; l++) x.visit_up(l);
  }
  x.store(a.u_top, x.U(Lc, x.cur(Lc)), 1 << Lc);
  x.bar("store", Lc);
  x.dump();
}

// f cascade: each thread restricts 2^S consecutive rows of one column down S
// levels with a binary-counter stack, pairing (left, right) exactly like
// restrict() applied level by level (stencils.py:39-47).
template <typename T, int S, typename M = T>
__global__ void k_cascade(const M* __restrict__ src, CascadeDst<M> dst, i64 n_src, i64 ld, int B) {
  int r = blockIdx.x * 32 + threadIdx.x;
  if (r >= B) return;
  const i64 nblk = n_src >> S;
  for (i64 blk = (i64)blockIdx.y * blockDim.y + threadIdx.y; blk < nblk;
       blk += (i64)gridDim.y * blockDim.y) {
    const M* s = src + (blk << S) * ld + r;
    T stack[S];
#pragma unroll
    for (int i = 0; i < (1 << S); i++) {
      T v = cvt<T>(s[(i64)i * ld]);
#pragma unroll
      for (int k = 0; k < S; k++) {
        // at step i, level k+1 completes iff the low k+1 bits of i are all ones
        if (((i >> k) & 1) == 0) {
          stack[k] = v;
          break;
        }
        v = xmul(T(0.5), xadd(stack[k], v));
        i64 idx = ((blk << S) + i) >> (k + 1);
        dst.p[k][idx * ld + r] = cvt<M>(v);
      }
    }
  }
}

}  // namespace

template <typename T>
size_t coarse_smem_bytes(int m0, int Lc, int CW, int extra_cells) {
  i64 cells = 0;
  for (int l = m0; l <= Lc; l++) cells += (i64)1 << l;
  return (size_t)(3 * cells * CW + 3 * ((i64)1 << m0) + (i64)extra_cells * CW) * sizeof(T);
}

template <typename T, int CW, typename M>
static void launch_coarse_cw(const CoarseArgs<T, M>& a, size_t smem, cudaStream_t s) {
  const int granted = smem_optin((const void*)coarse_kernel<T, CW, M>);
  require(smem <= (size_t)granted, "coarse: shared memory budget exceeded");
  unsigned blocks = (unsigned)((a.B + CW - 1) / CW);
  coarse_kernel<T, CW, M><<<blocks, CNT, smem, s>>>(a);
}

template <typename T, typename M>
static void launch_coarse_tm(const CoarseArgs<T, M>& a, cudaStream_t s) {
  require(a.Lc >= a.m0 && a.Lc < 31, "coarse: bad cutoff");
  size_t smem = coarse_smem_bytes<T>(a.m0, a.Lc, a.CW,
                                     (a.pj ? 1 << a.Lc : 0) +
                                         (a.fo ? (1 << (a.Lc + 1)) - (1 << a.m0) : 0));
  require(!a.fo || (a.mode == 0 && a.Lc == a.m), "coarse: on-chip cascade needs the whole solve");
  require(smem <= 227 * 1024, "coarse: shared memory budget exceeded");
  switch (a.CW) {
    case 1: launch_coarse_cw<T, 1>(a, smem, s); break;
    case 2: launch_coarse_cw<T, 2>(a, smem, s); break;
    case 4: launch_coarse_cw<T, 4>(a, smem, s); break;
    case 8: launch_coarse_cw<T, 8>(a, smem, s); break;
    case 16: launch_coarse_cw<T, 16>(a, smem, s); break;
    case 32: launch_coarse_cw<T, 32>(a, smem, s); break;
    default: require(false, "coarse: column group must be a power of two <= 32");
  }
  check_launch("coarse_kernel");
}

template <typename T>
void launch_coarse(const CoarseArgs<T>& a, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value) {
    if (a.f64_arith) {  // fp64 levels on chip over the fp32 fields
      CoarseArgs<double, float> b;
      b.m0 = a.m0, b.Lc = a.Lc, b.m = a.m, b.n_sr = a.n_sr, b.mode = a.mode;
      b.CW = a.CW, b.B = a.B, b.ld = a.ld;
      for (int l = 0; l < 32; l++) {
        b.W[l] = a.W[l];
        b.b[l] = a.b[l];
        b.forig[l] = a.forig[l];
        b.lgW[l] = a.lgW[l];
        b.off[l] = a.off[l];
        b.slen[l] = a.slen[l];
      }
      b.f_top = a.f_top;
      b.u_top = a.u_top;
      b.omega = a.omega;
      b.kz.proj_diag = (double)a.kz.proj_diag;
      b.kz.recip = (double)a.kz.recip;
      b.kz.pow2 = a.kz.pow2;
      b.trace = a.trace;
      b.fields = a.fields, b.scratch = a.scratch, b.nw = a.nw, b.pj = a.pj, b.fo = a.fo;
      require(!b.fo, "coarse: fp64 arithmetic on fp32 fields needs the f cascade in HBM");
      launch_coarse_tm(b, s);
      return;
    }
  }
  launch_coarse_tm(a, s);
}

template <typename T>
void launch_cascade(const T* src, i64 n_src, const CascadeDst<T>& dst, i64 ld, int B,
                    cudaStream_t s) {
  require(dst.levels >= 1 && dst.levels <= 6, "cascade: 1..6 levels per launch");
  require((n_src >> dst.levels) >= 1, "cascade: too many levels");
  dim3 block(32, 4);
  i64 blocks_y = ((n_src >> dst.levels) + 3) / 4;
  if (blocks_y > 16384) blocks_y = 16384;
  dim3 grid((unsigned)((B + 31) / 32), (unsigned)blocks_y);
  switch (dst.levels) {
    case 1: k_cascade<T, 1><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 2: k_cascade<T, 2><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 3: k_cascade<T, 3><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 4: k_cascade<T, 4><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 5: k_cascade<T, 5><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    default: k_cascade<T, 6><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
  }
  check_launch("cascade");
}

void launch_cascade_f64arith(const float* src, i64 n_src, const CascadeDst<float>& dst, i64 ld,
                             int B, cudaStream_t s) {
  require(dst.levels >= 1 && dst.levels <= 6, "cascade: 1..6 levels per launch");
  require((n_src >> dst.levels) >= 1, "cascade: too many levels");
  dim3 block(32, 4);
  i64 blocks_y = ((n_src >> dst.levels) + 3) / 4;
  if (blocks_y > 16384) blocks_y = 16384;
  dim3 grid((unsigned)((B + 31) / 32), (unsigned)blocks_y);
  switch (dst.levels) {
    case 1: k_cascade<double, 1, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 2: k_cascade<double, 2, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 3: k_cascade<double, 3, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 4: k_cascade<double, 4, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    case 5: k_cascade<double, 5, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
    default: k_cascade<double, 6, float><<<grid, block, 0, s>>>(src, dst, n_src, ld, B); break;
  }
  check_launch("cascade");
}

template size_t coarse_smem_bytes<double>(int, int, int, int);
template size_t coarse_smem_bytes<float>(int, int, int, int);
template void launch_coarse<double>(const CoarseArgs<double>&, cudaStream_t);
template void launch_coarse<float>(const CoarseArgs<float>&, cudaStream_t);
template void launch_cascade<double>(const double*, i64, const CascadeDst<double>&, i64, int, cudaStream_t);
template void launch_cascade<float>(const float*, i64, const CascadeDst<float>&, i64, int, cudaStream_t);

}  // namespace fmgsr
