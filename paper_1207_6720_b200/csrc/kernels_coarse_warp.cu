// kernels_coarse_warp.cu -- the coarse end of the hierarchy, one warp per RHS.
//
// Below the cutoff Lc every level visit is microseconds of latency-bound work.
// Right-hand sides are independent, so each CTA of NW warps (NW = 1, 2, 4, 8)
// owns ONE column and runs all visits of levels m0..Lc for it out of its own
// slice of shared memory; the 32 NW threads split each phase (patch chains,
// restriction rows, prolongation rows), one chain per thread on the deepest
// level, and phases are separated by __syncwarp() (NW = 1) or a barrier of
// the column's own CTA -- columns never wait for one another.
//   mode 0 (coarse FMG): the coarsest solve and FMG steps m0+1..Lc
//                        (reference cycles.py:178-199 for those levels);
//   mode 1 (V segment) : for a step t > Lc, the part of its V-cycle below
//                        Lc+1 (cycles.py:95-134).
// Layout per level: u0, u1, f, each n_l + n_l/W_l cells -- one pad cell per
// patch, so lane p reading cell p*W + i of its patch hits bank pair
// (p*(W+1) + i) mod 16: conflict-free in each half-warp (W + 1 is odd).
// Smoothers: ns = 1 (one forward chain with the visit's prologue just in time)
// and ns = 2 (forward chain, then Kaczmarz + backward chain over the forward
// values: owned cells in place in the output level, buffer cells and the two
// frozen window ends in a per-chain scratch of 2b + 2 cells), linear or the
// nonlinear Newton-GS.  Every operator is the exact-order device function of
// the grid kernels, so results stay bit-identical to the reference / oracle.
#include <cmath>
#include <cstdio>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

namespace {

__device__ __forceinline__ double p2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

template <typename T, bool NS2, bool NL, int NW>
struct Warp {
  static constexpr int NT = 32 * NW;  // threads per column
  const CoarseArgs<T>& a;
  T* base;      // this warp's slice
  T* scr;       // ns2 scratch (per chain 2b+2 cells, lane-strided) / Newton work
  T* dfac;      // linear direct factor d[n0], e[n0]
  T* efac;
  int lane;  // thread index within the column's CTA (0 .. NT-1)
  unsigned curmask;
  __device__ Warp(const CoarseArgs<T>& args) : a(args) {}

  __device__ __forceinline__ int N(int l) const { return 1 << l; }
  __device__ __forceinline__ int pd(int l, int c) const { return c + (c >> a.lgW[l]); }
  __device__ __forceinline__ T* U(int l, int w) const { return base + a.off[l] + w * a.slen[l]; }
  __device__ __forceinline__ T* F(int l) const { return U(l, 2); }
  __device__ __forceinline__ int cur(int l) const { return (curmask >> l) & 1; }
  __device__ __forceinline__ void flip(int l) { curmask ^= 1u << l; }
  __device__ __forceinline__ bool sr(int l) const { return l > a.m - a.n_sr; }
  // FMGSR_COARSE_TRACE=1: thread 0 of CTA 0 stamps the clock at every phase
  // barrier and prints the deltas at exit (phase-latency profiling)
  long long* ts = nullptr;
  int nts = 0;
  __device__ __forceinline__ void sync() {
    if (NW == 1) __syncwarp();
    else __syncthreads();
    if (ts && lane == 0 && nts < 128) ts[nts++] = clock64();
  }
  __device__ void dump() const {
    if (ts && lane == 0)
      for (int i = 1; i < nts; i++) printf("coarse-warp-trace %d %lld\n", i, ts[i] - ts[i - 1]);
  }

  __device__ GsCoef<T> coef(int l) const {
    GsCoef<T> gc;
    gc.inv_h2 = (T)p2d(2 * l);
    gc.rdiag = (T)p2d(-(2 * l + 1));
    gc.diag_b = xmul(T(3), gc.inv_h2);
    gc.omega = (T)a.omega;
    gc.diag_i = xmul(T(2), gc.inv_h2);
    return gc;
  }

  // ---- global <-> shared (one column, padded layout) --------------------------
  __device__ void load(T* dst, const T* src, int l) {
    const int n = N(l);
    for (int i = lane; i < n; i += NT) cp_async(dst + pd(l, i), src + (i64)i * a.ld);
    cp_commit();
    cp_wait<0>();
    sync();
  }
  __device__ void store(T* dst, const T* src, int l) {
    const int n = N(l);
    for (int i = lane; i < n; i += NT) dst[(i64)i * a.ld] = src[pd(l, i)];
  }

  // ---- prologue sources (value of the smoother input at fine cell x) ----------
  // prolong_fmg row x (stencils.py:67-105) from coarse level lc = l-1
  __device__ __forceinline__ T fmg(int l, const T* s, int x) const {
    const int nc = N(l - 1), nf = 2 * nc, lc = l - 1;
#define C(k) s[pd(lc, (k))]
    T v;
    if (x >= 4 && x < nf - 4) {
      const int q = x >> 1;
      if ((x & 1) == 0)
        v = xsub(xadd(xadd(xmul(T(-5), C(q - 2)), xmul(T(35), C(q - 1))), xmul(T(105), C(q))),
                 xmul(T(7), C(q + 1)));
      else
        v = xsub(xadd(xadd(xmul(T(-7), C(q - 1)), xmul(T(105), C(q))), xmul(T(35), C(q + 1))),
                 xmul(T(5), C(q + 2)));
    } else if (x == 0) v = xsub(xmul(T(70), C(0)), xmul(T(2), C(1)));
    else if (x == 1) v = xsub(xadd(xmul(T(112), C(0)), xmul(T(35), C(1))), xmul(T(5), C(2)));
    else if (x == 2) v = xsub(xadd(xmul(T(40), C(0)), xmul(T(105), C(1))), xmul(T(7), C(2)));
    else if (x == 3)
      v = xsub(xadd(xadd(xmul(T(-7), C(0)), xmul(T(105), C(1))), xmul(T(35), C(2))), xmul(T(5), C(3)));
    else if (x == nf - 4)
      v = xsub(xadd(xadd(xmul(T(-7), C(nc - 1)), xmul(T(105), C(nc - 2))), xmul(T(35), C(nc - 3))),
               xmul(T(5), C(nc - 4)));
    else if (x == nf - 3)
      v = xsub(xadd(xmul(T(40), C(nc - 1)), xmul(T(105), C(nc - 2))), xmul(T(7), C(nc - 3)));
    else if (x == nf - 2)
      v = xsub(xadd(xmul(T(112), C(nc - 1)), xmul(T(35), C(nc - 2))), xmul(T(5), C(nc - 3)));
    else v = xsub(xmul(T(70), C(nc - 1)), xmul(T(2), C(nc - 2)));
#undef C
    return xmul(v, T(0.0078125));
  }
  // u[x] + P(uH - R u)[x] (cycles.py:120-121, stencils.py:39-64)
  __device__ __forceinline__ T corr(int l, const T* u, const T* uH, int x) const {
    const int nf = N(l), nc = nf >> 1, lc = l - 1;
    auto cc = [&](int j) {
      return xsub(uH[pd(lc, j)], xmul(T(0.5), xadd(u[pd(l, 2 * j)], u[pd(l, 2 * j + 1)])));
    };
    T p;
    if (x == 0) p = xmul(T(0.5), cc(0));
    else if (x == nf - 1) p = xmul(T(0.5), cc(nc - 1));
    else if (x & 1) {
      const int j = (x - 1) >> 1;
      p = xmul(T(0.25), xadd(xmul(T(3), cc(j)), cc(j + 1)));
    } else {
      const int j = (x - 2) >> 1;
      p = xmul(T(0.25), xadd(cc(j), xmul(T(3), cc(j + 1))));
    }
    return xadd(u[pd(l, x)], p);
  }
  // SRC: 0 LOAD (u), 1 CORR (u, uH), 2 FMG (uH)
  template <int SRC>
  __device__ __forceinline__ T raw(int l, const T* u, const T* uH, int x) const {
    if (SRC == 0) return u[pd(l, x)];
    if (SRC == 1) return corr(l, u, uH, x);
    return fmg(l, uH, x);
  }
  // first Kaczmarz pass just in time: pairs in [wlo, whi) projected onto uc
  template <int SRC, bool CR>
  __device__ __forceinline__ T val(int l, const T* u, const T* uH, int x, int wlo, int whi) const {
    if (!CR) return raw<SRC>(l, u, uH, x);
    const int j = x >> 1;
    if (j < wlo || j >= whi) return raw<SRC>(l, u, uH, x);
    T p = raw<SRC>(l, u, uH, 2 * j), q = raw<SRC>(l, u, uH, 2 * j + 1);
    kaczmarz_pair(p, q, uH[pd(l - 1, j)], a.kz);
    return (x & 1) ? q : p;
  }
  __device__ __forceinline__ T gs(const GsCoef<T>& gc, int i, int n, T uL, T u, T uR, T f) const {
    // (the split-division interior Newton step, gs_int_nl, measured slower here:
    //  247 vs 227 us per V segment at config 3)
    return NL ? gs_cell_nl(gc, i, n, uL, u, uR, f) : gs_cell(gc, i, n, uL, u, uR, f);
  }

  // ---- patch smoother: out (level l) = S(input given by SRC / CR) -------------------
  template <int SRC, bool CR>
  __device__ void smooth(int l, const T* u, const T* uH, const T* f, T* out) {
    const int n = N(l), W = (int)a.W[l], b = (int)a.b[l], P = n / W;
    const GsCoef<T> gc = coef(l);
    for (int p = lane; p < P; p += NT) {
      const int os = p * W, oe = os + W;
      const int ws = os - b > 0 ? os - b : 0;
      const int we = oe + b < n ? oe + b : n;
      const int wlo = ws >> 1, whi = we >> 1;
      T uL = ws > 0 ? val<SRC, CR>(l, u, uH, ws - 1, wlo, whi) : T(0);
      T cu = val<SRC, CR>(l, u, uH, ws, wlo, whi);
      T nx = ws + 1 < n ? val<SRC, CR>(l, u, uH, ws + 1, wlo, whi) : T(0);
      if (!NS2) {
        // ns = 1: the chain stops at the owned end
        for (int i = ws; i < oe; i++) {
          const T nn = i + 2 < n ? val<SRC, CR>(l, u, uH, i + 2, wlo, whi) : T(0);
          const T v = gs(gc, i, n, uL, cu, nx, f[pd(l, i)]);
          if (i >= os) out[pd(l, i)] = v;
          uL = v;
          cu = nx;
          nx = nn;
        }
      } else {
        // scratch slots (lane-strided): 0 = frozen ws-1, 1..os-ws = left buffer,
        // then the right buffer oe..we-1, last = frozen we
        T* sc = scr + lane;
        const int nl = os - ws, nr = we - oe;
        auto sidx = [&](int x) -> int {
          return x < ws ? 0 : x < os ? 1 + (x - ws) : 1 + nl + (x - oe);
        };
        sc[0] = uL;  // first-pass value of ws-1 (projected when its pair is in range)
        for (int i = ws; i < we; i++) {
          const T nn = i + 2 < n ? val<SRC, CR>(l, u, uH, i + 2, wlo, whi) : T(0);
          const T v = gs(gc, i, n, uL, cu, nx, f[pd(l, i)]);
          if (i >= os && i < oe) out[pd(l, i)] = v;
          else sc[NT * sidx(i)] = v;
          uL = v;
          cu = nx;
          nx = nn;
        }
        if (we < n) sc[NT * (1 + nl + nr)] = cu;  // raw value of we (pair we/2 never projected)
        // backward: second Kaczmarz pass on the forward values, just in time
        auto fv = [&](int x) -> T {
          return (x >= os && x < oe) ? out[pd(l, x)] : x >= we ? sc[NT * (1 + nl + nr)] : sc[NT * sidx(x)];
        };
        auto fv2 = [&](int x) -> T {  // pass-2 value of x (its pair projected if in range)
          if (!CR) return fv(x);
          const int j = x >> 1;
          if (j < wlo || j >= whi) return fv(x);
          T p = fv(2 * j), q = fv(2 * j + 1);
          kaczmarz_pair(p, q, uH[pd(l - 1, j)], a.kz);
          return (x & 1) ? q : p;
        };
        T uR = we < n ? fv(we) : T(0);
        T c2 = fv2(we - 1);
        for (int i = we - 1; i >= ws; i--) {
          const T pv = i - 1 >= 0 ? fv2(i - 1) : T(0);
          const T v = gs(gc, i, n, pv, c2, uR, f[pd(l, i)]);
          if (i >= os && i < oe) out[pd(l, i)] = v;
          uR = v;
          c2 = pv;
        }
      }
    }
    sync();
  }

  // ---- restriction + tau (stencils.py:108-125; nonlinear: N u = L u + u^3) ------
  __device__ void restrict_tau(int l, const T* u, const T* f, T* uH, T* fH) {
    const int nf = N(l), nc = nf >> 1, lc = l - 1;
    const T ih = (T)p2d(2 * l), iH = (T)p2d(2 * lc);
    auto U_ = [&](int i) { return u[pd(l, i)]; };
    auto ru = [&](int k) { return xmul(T(0.5), xadd(U_(2 * k), U_(2 * k + 1))); };
    auto lu = [&](int i) {
      T s;
      if (i == 0) s = xsub(xmul(T(3), U_(0)), U_(1));
      else if (i == nf - 1) s = xsub(xmul(T(3), U_(nf - 1)), U_(nf - 2));
      else s = xsub(xsub(xmul(T(2), U_(i)), U_(i - 1)), U_(i + 1));
      T v = xmul(s, ih);
      if (NL) v = xadd(v, cube(U_(i)));
      return v;
    };
    for (int j = lane; j < nc; j += NT) {
      const T Rj = ru(j);
      T LH;
      if (j == 0) LH = xmul(xsub(xmul(T(3), Rj), ru(1)), iH);
      else if (j == nc - 1) LH = xmul(xsub(xmul(T(3), Rj), ru(nc - 2)), iH);
      else LH = xmul(xsub(xsub(xmul(T(2), Rj), ru(j - 1)), ru(j + 1)), iH);
      if (NL) LH = xadd(LH, cube(Rj));
      const T RL = xmul(T(0.5), xadd(lu(2 * j), lu(2 * j + 1)));
      const T Rf = xmul(T(0.5), xadd(f[pd(l, 2 * j)], f[pd(l, 2 * j + 1)]));
      fH[pd(lc, j)] = xadd(Rf, xsub(LH, RL));
      if (uH) uH[pd(lc, j)] = Rj;
    }
    sync();
  }

  // ---- coarsest solve -------------------------------------------------------------
  // linear: LAPACK ?ptsv order (dptts2 with the dpttrf factor, smoothers.py:210-225)
  // nonlinear: linear first iterate + Newton steps (oracle orc_direct_solve_nl)
  __device__ void direct(T* u) {
    const int n = N(a.m0), l = a.m0;
    const T* f = F(l);
    if (lane == 0) {
      T prev = f[pd(l, 0)];
      u[pd(l, 0)] = prev;
      for (int i = 1; i < n; i++) {
        prev = xsub(f[pd(l, i)], xmul(prev, efac[i - 1]));
        u[pd(l, i)] = prev;
      }
      T nx = xdiv(prev, dfac[n - 1]);
      u[pd(l, n - 1)] = nx;
      for (int i = n - 2; i >= 0; i--) {
        nx = xsub(xdiv(u[pd(l, i)], dfac[i]), xmul(nx, efac[i]));
        u[pd(l, i)] = nx;
      }
      if (NL) {
        // Newton work arrays in this warp's scratch: d, e, r (n each)
        T* d = scr;
        T* e = scr + n;
        T* rr = scr + 2 * n;
        const T ih = (T)p2d(2 * l);
        auto UU = [&](int i) { return u[pd(l, i)]; };
        for (int it = 0; it < 10; it++) {
          for (int i = 0; i < n; i++) {
            T s;
            if (i == 0) s = xsub(xmul(T(3), UU(0)), UU(1));
            else if (i == n - 1) s = xsub(xmul(T(3), UU(n - 1)), UU(n - 2));
            else s = xsub(xsub(xmul(T(2), UU(i)), UU(i - 1)), UU(i + 1));
            const T ui = UU(i);
            const T Ni = xadd(xmul(s, ih), xmul(xmul(ui, ui), ui));
            rr[i] = xsub(f[pd(l, i)], Ni);
            d[i] = xadd(xmul(T((i == 0 || i == n - 1) ? 3 : 2), ih), xmul(T(3), xmul(ui, ui)));
            e[i] = -ih;
          }
          for (int i = 0; i < n - 1; i++) {
            const T ei = e[i];
            e[i] = xdiv(ei, d[i]);
            d[i + 1] = xsub(d[i + 1], xmul(e[i], ei));
          }
          for (int i = 1; i < n; i++) rr[i] = xsub(rr[i], xmul(rr[i - 1], e[i - 1]));
          rr[n - 1] = xdiv(rr[n - 1], d[n - 1]);
          for (int i = n - 2; i >= 0; i--) rr[i] = xsub(xdiv(rr[i], d[i]), xmul(rr[i + 1], e[i]));
          for (int i = 0; i < n; i++) u[pd(l, i)] = xadd(UU(i), rr[i]);
        }
      }
    }
    sync();
  }

  // ---- level visits ---------------------------------------------------------------
  __device__ void visit_top(int t) {  // u_t = Pi u_{t-1}, smooth, restrict + tau
    const int h = cur(t - 1);
    smooth<2, false>(t, nullptr, U(t - 1, h), F(t), U(t, 0));
    curmask &= ~(1u << t);
    restrict_tau(t, U(t, 0), F(t), U(t - 1, h ^ 1), F(t - 1));
    flip(t - 1);
  }
  __device__ void visit_down(int l) {
    const int c = cur(l);
    smooth<0, false>(l, U(l, c), nullptr, F(l), U(l, c ^ 1));
    flip(l);
    const int h = cur(l - 1);
    restrict_tau(l, U(l, c ^ 1), F(l), l - 1 == a.m0 ? nullptr : U(l - 1, h ^ 1), F(l - 1));
    if (l - 1 != a.m0) flip(l - 1);
  }
  __device__ void visit_direct() {
    const int c = cur(a.m0);
    direct(U(a.m0, c ^ 1));
    flip(a.m0);
  }
  __device__ void visit_up(int l) {
    const int c = cur(l);
    const T* uH = U(l - 1, cur(l - 1));
    if (sr(l)) smooth<2, true>(l, nullptr, uH, F(l), U(l, c ^ 1));
    else smooth<1, false>(l, U(l, c), uH, F(l), U(l, c ^ 1));
    flip(l);
  }
};

template <typename T, bool NS2, bool NL, int NW>
__global__ void __launch_bounds__(32 * NW) coarse_warp_kernel(const __grid_constant__ CoarseArgs<T> a) {
  extern __shared__ __align__(16) unsigned char cw_smem[];
  const int r = blockIdx.x;  // this warp's RHS column
  Warp<T, NS2, NL, NW> w(a);
  w.lane = threadIdx.x;
  __shared__ long long ts_s[128];
  if (a.trace && blockIdx.x == 0) w.ts = ts_s;
  w.base = reinterpret_cast<T*>(cw_smem);
  w.scr = w.base + a.fields;
  w.dfac = w.scr + a.scratch;
  w.efac = w.dfac + (1 << a.m0);
  w.curmask = 0;
  const int m0 = a.m0, Lc = a.Lc, n0 = 1 << m0;
  if (w.lane == 0) {  // dpttrf, as in k_direct_solve
    const T ih = (T)p2d(2 * m0);
    T* d = w.dfac;
    T* e = w.efac;
    for (int i = 0; i < n0; i++) d[i] = xmul(T(2), ih);
    d[0] = xmul(T(3), ih);
    d[n0 - 1] = xmul(T(3), ih);
    for (int i = 0; i < n0 - 1; i++) e[i] = -ih;
    for (int i = 0; i < n0 - 1; i++) {
      const T ei = e[i];
      e[i] = xdiv(ei, d[i]);
      d[i + 1] = xsub(d[i + 1], xmul(e[i], ei));
    }
  }
  const i64 col = r;
  if (a.mode == 0) {
    w.load(w.F(m0), a.forig[m0] + col, m0);
    w.visit_direct();
    for (int t = m0 + 1; t <= Lc; t++) {
      w.load(w.F(t), a.forig[t] + col, t);
      w.visit_top(t);
      for (int l = t - 1; l > m0; l--) w.visit_down(l);
      w.visit_direct();
      for (int l = m0 + 1; l <= t; l++) w.visit_up(l);
    }
  } else {
    w.load(w.U(Lc, 0), a.u_top + col, Lc);
    w.load(w.F(Lc), a.f_top + col, Lc);
    for (int l = Lc; l > m0; l--) w.visit_down(l);
    w.visit_direct();
    for (int l = m0 + 1; l <= Lc; l++) w.visit_up(l);
  }
  w.store(a.u_top + col, w.U(Lc, w.cur(Lc)), Lc);
  w.sync();
  w.dump();
}

}  // namespace

// Per-warp layout: fields of levels m0..Lc, then the ns2 / Newton scratch,
// then the direct-solve factor.  Fills a.lgW / a.off / a.slen / a.fields /
// a.scratch and returns the bytes of one warp's slice.
template <typename T>
size_t coarse_warp_layout(CoarseArgs<T>& a, bool ns2, bool nl) {
  i64 off = 0, scratch = 0;
  for (int l = a.m0; l <= a.Lc; l++) {
    const i64 n = (i64)1 << l, W = a.W[l] > 0 ? a.W[l] : n;
    int lg = 0;
    while (((i64)1 << (lg + 1)) <= W) lg++;
    a.lgW[l] = lg;
    i64 len = n + (n >> lg);
    len += len & 1;
    a.slen[l] = (int)len;
    a.off[l] = (int)off;
    off += 3 * len;
    if (ns2 && l > a.m0) {
      const i64 s = 32 * (i64)a.nw * (2 * a.b[l] + 2);
      if (s > scratch) scratch = s;
    }
  }
  if (nl && scratch < 3 * ((i64)1 << a.m0)) scratch = 3 * ((i64)1 << a.m0);
  a.fields = (int)off;
  a.scratch = (int)scratch;
  return (size_t)(off + scratch + 2 * ((i64)1 << a.m0)) * sizeof(T);
}

template <typename T>
void launch_coarse_warp(const CoarseArgs<T>& args, bool ns2, bool nl, cudaStream_t s) {
  CoarseArgs<T> a = args;
  require(a.Lc >= a.m0 && a.Lc < 31, "coarse: bad cutoff");
  const size_t smem = coarse_warp_layout(a, ns2, nl);
  require(smem <= 227 * 1024, "coarse: shared memory budget exceeded");
  auto go = [&](void (*kf)(const CoarseArgs<T>)) {
    const int g = smem_optin((const void*)kf);
    require(smem <= (size_t)g, "coarse: shared memory budget exceeded");
    kf<<<(unsigned)a.B, 32 * a.nw, smem, s>>>(a);
  };
#define CWK_NW(NS, NLV)                                      \
  switch (a.nw) {                                            \
    case 1: go(coarse_warp_kernel<T, NS, NLV, 1>); break;    \
    case 2: go(coarse_warp_kernel<T, NS, NLV, 2>); break;    \
    case 4: go(coarse_warp_kernel<T, NS, NLV, 4>); break;    \
    case 8: go(coarse_warp_kernel<T, NS, NLV, 8>); break;    \
    default: require(false, "coarse: warps per column must be 1, 2, 4 or 8"); \
  }
  if (ns2) {
    if (nl) {
      CWK_NW(true, true)
    } else {
      CWK_NW(true, false)
    }
  } else {
    if (nl) {
      CWK_NW(false, true)
    } else {
      CWK_NW(false, false)
    }
  }
#undef CWK_NW
  check_launch("coarse_warp_kernel");
}

template size_t coarse_warp_layout<double>(CoarseArgs<double>&, bool, bool);
template size_t coarse_warp_layout<float>(CoarseArgs<float>&, bool, bool);
template void launch_coarse_warp<double>(const CoarseArgs<double>&, bool, bool, cudaStream_t);
template void launch_coarse_warp<float>(const CoarseArgs<float>&, bool, bool, cudaStream_t);

}  // namespace fmgsr
