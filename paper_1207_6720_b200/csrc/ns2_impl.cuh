// ns2_impl.cuh -- the V(2,2) streaming smoother kernel (see kernels_ns2.cu)
// and its launch plumbing, instantiated per lane type in
// kernels_ns2_{d,f,v2d,v2f}.cu.
#pragma once

#include <cmath>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

namespace {

constexpr int NT2 = 128;
constexpr int D2 = 8;

template <typename T, bool NL>
__device__ __forceinline__ T gs2(const GsCoef<T>& c, i64 i, i64 n, T uL, T u, T uR, T f) {
  return NL ? gs_cell_nl(c, i, n, uL, u, uR, f) : gs_cell(c, i, n, uL, u, uR, f);
}
// interior cell (not a domain row)
template <typename T, bool NL, bool OMEGA1>
__device__ __forceinline__ T gs2i(const GsCoef<T>& c, T uL, T u, T uR, T f) {
  return NL ? gs_int_nl<T, OMEGA1>(c, uL, u, uR, f) : gs_int_o<T, OMEGA1>(c, uL, u, uR, f);
}

template <typename T>
struct Ns2Args {
  i64 n, ld, W, b, P, nc, p_begin, sld, srows;
  int B, nrg;
  GsCoef<T> gc;
  KzCoef<T> kz;
  T inv_H2;
  bool write_u;
  const T *u_src, *uH, *uc, *f;
  T *u_out, *scratch;
  T *uH_out, *fH_out, *E;  // fused restriction / tau (EPI)
  int* cnt;
};

// Restriction + tau epilogue of the BACKWARD sweep: the same coarse values
// and edge records as Epilogue (fmgsr_device.cuh) for pairs pushed in
// descending order.  Coarse cell c = j+1 is emitted when pair j arrives (it
// needs u at 2j+1 .. 2j+4); the right record is complete after two pairs, the
// left one after the last.  NL: operator values are N u = L u + u^3.
template <typename T, bool NL>
struct EpiRev {
  T ih, iH;
  bool left_dom, right_dom;
  T* uH_out;  // column-offset, may be null
  T* fH_out;  // column-offset
  i64 ld, nc;
  T p0, p1, R1, R2, Rf1, Lodd1;  // pair j+1 cells, R at j+1 / j+2, Rf at j+1, N u at 2j+3
  int cnt;
  EdgeRec<T> left, right;

  __device__ __forceinline__ T lu(T two_u, T um, T up) const {  // ((2u - um) - up) ih
    return xmul(xsub(xsub(two_u, um), up), ih);
  }
  __device__ __forceinline__ void push(i64 j, T a, T b, T f0, T f1, bool store) {
    const T Rj = xmul(T(0.5), xadd(a, b));
    const T Rfj = xmul(T(0.5), xadd(f0, f1));
    if (uH_out && store) uH_out[j * ld] = Rj;
    T Lodd = T(0);
    if (cnt == 0) {
      if (right_dom) {
        Lodd = xmul(xsub(xmul(T(3), b), a), ih);  // Lu[n-1]
        if (NL) Lodd = xadd(Lodd, cube(b));
      } else {
        right.v[0] = a;  // u[oe-2]
        right.v[1] = b;  // u[oe-1]
        right.v[4] = Rfj;
      }
    } else {
      T Lev = lu(xmul(T(2), p0), b, p1);  // Lu[2j+2]
      if (NL) Lev = xadd(Lev, cube(p0));
      if (cnt == 1 && !right_dom) {
        right.v[2] = Lev;  // Lu[oe-2]
        right.v[3] = Rj;   // Ru_{oe/2-2}
      } else {
        const i64 c = j + 1;
        T RL = xmul(T(0.5), xadd(Lev, Lodd1));
        T LH = (c == nc - 1) ? xmul(xsub(xmul(T(3), R1), Rj), iH)
                             : xmul(xsub(xsub(xmul(T(2), R1), Rj), R2), iH);
        if (NL) LH = xadd(LH, cube(R1));
        if (store) fH_out[c * ld] = xadd(Rf1, xsub(LH, RL));
      }
      Lodd = lu(xmul(T(2), b), a, p0);  // Lu[2j+1]
      if (NL) Lodd = xadd(Lodd, cube(b));
    }
    p0 = a;
    p1 = b;
    R2 = R1;
    R1 = Rj;
    Rf1 = Rfj;
    Lodd1 = Lodd;
    cnt++;
  }
  // steady state (cnt >= 2, c = j+1 < nc-1): pointers at uH[j], fH[j+1]
  T* puH;
  T* pfH;
  __device__ __forceinline__ void fast_begin(i64 j) {
    puH = uH_out ? uH_out + j * ld : nullptr;
    pfH = fH_out + (j + 1) * ld;
  }
  __device__ __forceinline__ void push_fast(T a, T b, T f0, T f1, bool store) {
    const T Rj = xmul(T(0.5), xadd(a, b));
    const T Rfj = xmul(T(0.5), xadd(f0, f1));
    if (uH_out && store) *puH = Rj;
    puH -= ld;
    T Lev = lu(xmul(T(2), p0), b, p1);
    if (NL) Lev = xadd(Lev, cube(p0));
    T RL = xmul(T(0.5), xadd(Lev, Lodd1));
    T LH = xmul(xsub(xsub(xmul(T(2), R1), Rj), R2), iH);
    if (NL) LH = xadd(LH, cube(R1));
    if (store) *pfH = xadd(Rf1, xsub(LH, RL));
    pfH -= ld;
    T Lodd = lu(xmul(T(2), b), a, p0);
    if (NL) Lodd = xadd(Lodd, cube(b));
    p0 = a;
    p1 = b;
    R2 = R1;
    R1 = Rj;
    Rf1 = Rfj;
    Lodd1 = Lodd;
    cnt++;
  }
  // after the first owned pair (os/2): close the domain start or build the left record
  __device__ __forceinline__ void finish(bool store) {
    if (left_dom) {
      T L0 = xmul(xsub(xmul(T(3), p0), p1), ih);  // Lu[0]
      if (NL) L0 = xadd(L0, cube(p0));
      T RL = xmul(T(0.5), xadd(L0, Lodd1));
      T LH = xmul(xsub(xmul(T(3), R1), R2), iH);
      if (NL) LH = xadd(LH, cube(R1));
      if (store) fH_out[0] = xadd(Rf1, xsub(LH, RL));
    } else {
      left.v[0] = p0;     // u[os]
      left.v[1] = p1;     // u[os+1]
      left.v[2] = Lodd1;  // Lu[os+1]
      left.v[3] = R2;     // Ru_{os/2+1}
      left.v[4] = Rf1;    // Rf_{os/2}
    }
  }
};

__device__ __forceinline__ i64 imax(i64 a, i64 b) { return a > b ? a : b; }
__device__ __forceinline__ i64 imin(i64 a, i64 b) { return a < b ? a : b; }

template <typename T, int SRC, bool CR, bool NL, bool OMEGA1, bool EPI>
__global__ void __launch_bounds__(NT2, sizeof(T) > 8 ? 2 : 4) ns2_kernel(const Ns2Args<T> a) {
  extern __shared__ __align__(16) unsigned char ns2_smem[];
  constexpr int R = SrcRows<SRC, CR>::R;
  constexpr int R2 = CR ? 5 : 4;  // backward rows: scratch(2) + f(2) [+ uc]
  const int lane = threadIdx.x & 31;
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 pl = gw / a.nrg;
  const int rg = (int)(gw - pl * a.nrg);
  if (pl >= a.P) return;
  const i64 p = a.p_begin + pl;
  const int r = rg * 32 + lane;
  const bool store = r < a.B;
  const int rr = store ? r : a.B - 1;
  const i64 n = a.n, ld = a.ld, sld = a.sld, nc = a.nc;
  const i64 os = p * a.W, oe = os + a.W;
  const i64 ws = os - a.b > 0 ? os - a.b : 0;
  const i64 we = oe + a.b < n ? oe + a.b : n;
  const i64 lo = ws > 0 ? ws - 1 : 0;
  const i64 hi = we < n ? we + 1 : n;
  const i64 wlo = ws >> 1, whi = we >> 1;
  // this lane's scratch column: window cell x at Sc[(x - lo) * sld]
  T* Sc = a.scratch + (pl * a.srows) * sld + r;
  T* ring = reinterpret_cast<T*>(ns2_smem) + threadIdx.x;
  const GsCoef<T> gc = a.gc;

  // ---------------- forward: prologue + Kaczmarz (JIT) + GS, spill ----------------
  PairSource<T, SRC, CR> src;
  src.u = a.u_src ? a.u_src + rr : nullptr;
  src.uH = a.uH ? a.uH + rr : nullptr;
  src.uc = a.uc ? a.uc + rr : nullptr;
  src.f = a.f + rr;
  src.ld = ld;
  src.nc = nc;
  src.kz = a.kz;
  src.wlo = wlo;
  src.whi = whi;
  src.qlo = 0;
  src.qhi = nc - 1;
  auto slot = [&](i64 x) { return ring + (i64)((x & (D2 - 1)) * R) * NT2; };
  const i64 qs = lo >> 1;        // first pair with a window cell
  const i64 qe = (hi - 1) >> 1;  // last pair with a window cell
  src.init(qs);
  T v0, v1, f0, f1;
  {
    Raw<T> rw = src.load(qs);
    src.make(qs, rw, v0, v1);
    f0 = rw.f0;
    f1 = rw.f1;
  }
  for (int k = 1; k < D2; k++) {
    src.template issue<NT2>(slot(qs + k), qs + k);
    cp_commit();
  }
  T uL = T(0);
  // fast pairs: both cells interior GS cells of the window, next pair made by make_fast
  i64 qf_lo = (imax(ws, 1) + 1) >> 1;
  i64 qf_hi = (imin(we - 1, n - 2) - 1) >> 1;
  if (SRC == SRC_FMG) {
    qf_lo = imax(qf_lo, 1);
    qf_hi = imin(qf_hi, nc - 4);
  } else if (SRC == SRC_CORR) {
    qf_hi = imin(qf_hi, nc - 3);
  }
  if (CR) {
    qf_lo = imax(qf_lo, wlo - 1);
    qf_hi = imin(qf_hi, whi - 2);
  }
  auto fwd_slow = [&](i64 q) {
    cp_wait<D2 - 2>();
    Raw<T> rw = src.template fetch<NT2>(slot(q + 1));
    src.template issue<NT2>(slot(q), q + D2);
    cp_commit();
    T w0, w1;
    src.make(q + 1, rw, w0, w1);
    const i64 i0 = 2 * q, i1 = i0 + 1;
    if (i0 >= lo && i0 < hi) {
      T x = v0;
      if (i0 >= ws && i0 < we) x = gs2<T, NL>(gc, i0, n, uL, v0, v1, f0);
      Sc[(i0 - lo) * sld] = x;
      uL = x;
    }
    if (i1 >= lo && i1 < hi) {
      T x = v1;
      if (i1 >= ws && i1 < we) x = gs2<T, NL>(gc, i1, n, uL, v1, w0, f1);
      Sc[(i1 - lo) * sld] = x;
      uL = x;
    }
    v0 = w0;
    v1 = w1;
    f0 = rw.f0;
    f1 = rw.f1;
  };
  i64 q = qs;
  for (; q <= qe && q < qf_lo; q++) fwd_slow(q);
  {
    // fast step on ring slots sn (pair q+1) / si (pair q, refilled with q+D2);
    // pointer-stepped unclamped issue while pair q+D2's rows all exist
    constexpr int OFF = SRC == SRC_FMG ? 2 : SRC == SRC_CORR ? 1 : 0;
    const i64 q_if = imin(qf_hi, nc - 1 - D2 - OFF);
    T* sp = Sc + (2 * q - lo) * sld;
    auto fwd_fast = [&](i64 qq, int sn, int si, bool unclamped) {
      cp_wait<D2 - 2>();
      Raw<T> rw = src.template fetch<NT2>(ring + sn * R * NT2);
      if (unclamped) src.template issue_fast<NT2>(ring + si * R * NT2);
      else src.template issue<NT2>(ring + si * R * NT2, qq + D2);
      cp_commit();
      T w0, w1;
      src.make_fast(rw, w0, w1);
      const T x0 = gs2i<T, NL, OMEGA1>(gc, uL, v0, v1, f0);
      sp[0] = x0;
      const T x1 = gs2i<T, NL, OMEGA1>(gc, x0, v1, w0, f1);
      sp[sld] = x1;
      sp += 2 * sld;
      uL = x1;
      v0 = w0;
      v1 = w1;
      f0 = rw.f0;
      f1 = rw.f1;
    };
    if (q <= q_if) {
      src.fast_ptrs(q + D2);
      for (; q <= q_if && (q & (D2 - 1)) != 0; q++) fwd_fast(q, (int)((q + 1) & (D2 - 1)), (int)(q & (D2 - 1)), true);
      for (; q + (D2 - 1) <= q_if; q += D2) {
#pragma unroll
        for (int k = 0; k < D2; k++) fwd_fast(q + k, (k + 1) & (D2 - 1), k, true);
      }
      for (; q <= q_if; q++) fwd_fast(q, (int)((q + 1) & (D2 - 1)), (int)(q & (D2 - 1)), true);
    }
    for (; q <= qf_hi; q++) fwd_fast(q, (int)((q + 1) & (D2 - 1)), (int)(q & (D2 - 1)), false);
  }
  for (; q <= qe; q++) fwd_slow(q);
  cp_wait<0>();
  __syncwarp();

  // ---------------- backward: Kaczmarz (JIT) + GS over the spilled window ----------
  // pair j rows: Sc[2j], Sc[2j+1] (this lane's column), f[2j], f[2j+1], uc[j]
  const T* fcol = a.f + rr;
  const T* ucol = CR ? (SRC == SRC_FMG ? a.uH + rr : a.uc + rr) : nullptr;
  auto slot2 = [&](i64 x) { return ring + (i64)((x & (D2 - 1)) * R2) * NT2; };
  const i64 jt = (we - 1) >> 1;  // first pair of the backward sweep
  const i64 jb = lo >> 1;        // last pair (holds ws-1 or ws)
  auto issue2 = [&](i64 j) {
    T* s = slot2(j);
    if (j > jb && 2 * j + 1 < hi) {  // rows inside the window column: no clamping
      const T* sp = Sc + (2 * j - lo) * sld;
      cp_async(s, sp);
      cp_async(s + NT2, sp + sld);
      const T* fp = fcol + (2 * j) * ld;
      cp_async(s + 2 * NT2, fp);
      cp_async(s + 3 * NT2, fp + ld);
      if (CR) cp_async(s + 4 * NT2, ucol + j * ld);
      return;
    }
    const i64 jj = j < jb ? jb : j;
    // window cells outside [lo, hi) are never read; clamp rows into the column
    i64 x0 = 2 * jj, x1 = 2 * jj + 1;
    x0 = x0 < lo ? lo : (x0 >= hi ? hi - 1 : x0);
    x1 = x1 < lo ? lo : (x1 >= hi ? hi - 1 : x1);
    cp_async(s, Sc + (x0 - lo) * sld);
    cp_async(s + NT2, Sc + (x1 - lo) * sld);
    i64 f0r = 2 * jj, f1r = 2 * jj + 1;
    f1r = f1r >= n ? n - 1 : f1r;
    cp_async(s + 2 * NT2, fcol + f0r * ld);
    cp_async(s + 3 * NT2, fcol + f1r * ld);
    if (CR) cp_async(s + 4 * NT2, ucol + (jj >= nc ? nc - 1 : jj) * ld);
  };
  for (int k = 0; k < D2 - 1; k++) {
    issue2(jt - k);
    cp_commit();
  }
  // projected (second Kaczmarz pass) values of pair j
  auto pair_vals = [&](i64 j, T& a0, T& a1, T& g0, T& g1) {
    cp_wait<D2 - 2>();
    const T* s = slot2(j);
    a0 = s[0];
    a1 = s[NT2];
    g0 = s[2 * NT2];
    g1 = s[3 * NT2];
    if (CR && j >= wlo && j < whi) kaczmarz_pair(a0, a1, s[4 * NT2], a.kz);
    issue2(j - (D2 - 1));
    cp_commit();
  };
  T a0, a1, g0, g1;
  pair_vals(jt, a0, a1, g0, g1);
  // frozen right neighbour of the window (never projected: pair we>>1 = whi)
  T uR = T(0);
  if (we < n) uR = (we & 1) ? a1 : Sc[(we - lo) * sld];
  const bool wu = store && (!EPI || a.write_u);
  T* out = a.u_out + r;
  EpiRev<T, NL> ep;
  if (EPI) {
    ep.ih = gc.inv_h2;
    ep.iH = a.inv_H2;
    ep.left_dom = os == 0;
    ep.right_dom = oe == n;
    ep.uH_out = a.uH_out ? a.uH_out + r : nullptr;
    ep.fH_out = a.fH_out + r;
    ep.ld = ld;
    ep.nc = nc;
    ep.cnt = 0;
    ep.p0 = ep.p1 = ep.R1 = ep.R2 = ep.Rf1 = ep.Lodd1 = T(0);
  }
  auto bwd_slow = [&](i64 j) {
    const i64 i1 = 2 * j + 1, i0 = 2 * j;
    T b0 = T(0), b1 = T(0), h0 = T(0), h1 = T(0);
    if (j - 1 >= jb) pair_vals(j - 1, b0, b1, h0, h1);
    T x1 = T(0), x0 = T(0);
    if (i1 >= ws && i1 < we) {
      const T v = gs2<T, NL>(gc, i1, n, a0, a1, uR, g1);
      if (wu && i1 >= os && i1 < oe) out[i1 * ld] = v;
      uR = v;
      x1 = v;
    }
    // cell 2j: its left neighbour 2j-1 is the second cell of pair j-1
    if (i0 >= ws && i0 < we) {
      const T v = gs2<T, NL>(gc, i0, n, b1, a0, uR, g0);
      if (wu && i0 >= os && i0 < oe) out[i0 * ld] = v;
      uR = v;
      x0 = v;
    }
    if (EPI && i0 >= os && i1 < oe) ep.push(j, x0, x1, g0, g1, store);
    a0 = b0;
    a1 = b1;
    g0 = h0;
    g1 = h1;
  };
  // fast pairs: both cells owned interior cells, pair j-1 exists
  const i64 jf_hi = imin((imin(oe - 1, n - 2) - 1) >> 1, EPI ? (oe >> 1) - 3 : nc);
  const i64 jf_lo = imax((imax(os, 1) + 1) >> 1, jb + 1);
  i64 j = jt;
  for (; j >= jb && j > jf_hi; j--) bwd_slow(j);
  {
    // fast step: pair j-1 from slot sj (projected when in the Kaczmarz range),
    // slot si (pair j, consumed) refilled with pair j-D2 -- pointer-stepped
    // (sp2/fp2/up2 at pair j-D2) while that pair lies inside the window
    T* op = out + (2 * j) * ld;
    if (EPI) ep.fast_begin(j);
    const i64 g0i = j - D2;
    const T* sp2 = Sc + (2 * g0i - lo) * sld;
    const T* fp2 = fcol + (2 * g0i) * ld;
    const T* up2 = CR ? ucol + g0i * ld : nullptr;
    auto bwd_fast = [&](i64 jj, int sj, int si, bool unclamped) {
      cp_wait<D2 - 2>();
      const T* s2 = ring + sj * R2 * NT2;
      T b0 = s2[0], b1 = s2[NT2], h0 = s2[2 * NT2], h1 = s2[3 * NT2];
      if (CR && jj - 1 >= wlo && jj - 1 < whi) kaczmarz_pair(b0, b1, s2[4 * NT2], a.kz);
      if (unclamped) {
        T* d = ring + si * R2 * NT2;
        cp_async(d, sp2);
        cp_async(d + NT2, sp2 + sld);
        cp_async(d + 2 * NT2, fp2);
        cp_async(d + 3 * NT2, fp2 + ld);
        if (CR) cp_async(d + 4 * NT2, up2);
      } else {
        issue2(jj - D2);
      }
      cp_commit();
      sp2 -= 2 * sld;
      fp2 -= 2 * ld;
      if (CR) up2 -= ld;
      const T x1 = gs2i<T, NL, OMEGA1>(gc, a0, a1, uR, g1);
      const T x0 = gs2i<T, NL, OMEGA1>(gc, b1, a0, x1, g0);
      if (wu) {
        op[ld] = x1;
        op[0] = x0;
      }
      op -= 2 * ld;
      if (EPI) ep.push_fast(x0, x1, g0, g1, store);
      uR = x0;
      a0 = b0;
      a1 = b1;
      g0 = h0;
      g1 = h1;
    };
    // unclamped refills while pair j-D2 > jb
    const i64 j_if = imax(jf_lo, jb + D2 + 1);
    for (; j >= j_if && (j & (D2 - 1)) != D2 - 1; j--)
      bwd_fast(j, (int)((j - 1) & (D2 - 1)), (int)(j & (D2 - 1)), true);
    for (; j - (D2 - 1) >= j_if; j -= D2) {
#pragma unroll
      for (int k = 0; k < D2; k++) bwd_fast(j - k, (D2 - 2 - k) & (D2 - 1), D2 - 1 - k, true);
    }
    for (; j >= j_if; j--) bwd_fast(j, (int)((j - 1) & (D2 - 1)), (int)(j & (D2 - 1)), true);
    for (; j >= jf_lo; j--) bwd_fast(j, (int)((j - 1) & (D2 - 1)), (int)(j & (D2 - 1)), false);
  }
  for (; j >= jb; j--) bwd_slow(j);
  cp_wait<0>();
  if (EPI) {
    ep.finish(store);
    const i64 ldE = (i64)a.nrg * 32;
    edge_arrive2<T, NL>(a.E, a.cnt, ldE, a.nrg, lane, rg, r, store, ep.fH_out, ld, ep.ih, ep.iH,
                        !ep.left_dom, p, ep.left, os, !ep.right_dom, p + 1, ep.right, oe);
  }
}

}  // namespace

template <typename TV, typename T0>
void ns2_fill_launch(const Ns2Desc<T0>& d, cudaStream_t s) {
  using T = TV;  // lane type: T0 or V2<T0>
  constexpr int C = LaneCols<TV>::value;
  auto cv = [](const T0* p) { return reinterpret_cast<const TV*>(p); };
  auto mv = [](T0* p) { return reinterpret_cast<TV*>(p); };
  Ns2Args<T> a;
  a.n = d.n;
  a.ld = d.ld / C;
  a.B = d.B / C;
  a.nrg = (a.B + 31) / 32;
  a.W = d.W;
  a.b = d.b;
  a.nc = d.n / 2;
  a.P = d.n / d.W;
  a.p_begin = 0;
  a.srows = d.W + 2 * d.b + 2;
  a.sld = (i64)a.nrg * 32;
  require(d.sld / C >= a.sld, "ns2: scratch stride too small");
  a.sld = d.sld / C;
  int k = level_of(d.n);
  double ih = pow4(k);
  a.gc.inv_h2 = (T)ih;
  a.gc.rdiag = (T)(1.0 / (2.0 * ih));
  a.gc.diag_b = (T)(3.0 * ih);
  a.gc.omega = (T)d.omega;
  a.gc.diag_i = (T)(2.0 * ih);
  a.kz.proj_diag = (T)d.proj_diag;
  int e;
  a.kz.pow2 = std::frexp(d.proj_diag, &e) == 0.5;
  a.kz.recip = (T)(a.kz.pow2 ? std::ldexp(1.0, 1 - e) : 1.0 / d.proj_diag);
  a.u_src = cv(d.u_src);
  a.uH = cv(d.uH);
  a.uc = cv(d.uc);
  a.f = cv(d.f);
  a.u_out = mv(d.u_out);
  a.scratch = mv(d.scratch);
  a.inv_H2 = (T)pow4(k - 1);
  a.write_u = d.write_u;
  a.uH_out = mv(d.uH_out);
  a.fH_out = mv(d.fH_out);
  a.E = mv(d.E);
  a.cnt = d.cnt;
  const i64 blocks = (a.P * a.nrg + NT2 / 32 - 1) / (NT2 / 32);
  const size_t smem = (size_t)D2 * 6 * NT2 * sizeof(T);  // max(R, R2) rows per slot (48 / 96 KB)
  const bool om1 = d.omega == 1.0;
  auto go = [&](void (*kf)(const Ns2Args<T>)) {
    if (smem > 48 * 1024)
      require(smem <= (size_t)smem_optin((const void*)kf), "ns2: shared memory budget exceeded");
    kf<<<(unsigned)blocks, NT2, smem, s>>>(a);
  };
#define NS2_OM(SRCV, CRV, NLV, EPIV)                   \
  if (om1) go(ns2_kernel<T, SRCV, CRV, NLV, true, EPIV>); \
  else go(ns2_kernel<T, SRCV, CRV, NLV, false, EPIV>);
#define NS2_NL(SRCV, CRV, EPIV)                 \
  if (d.nonlinear) {                            \
    NS2_OM(SRCV, CRV, true, EPIV)               \
  } else {                                      \
    NS2_OM(SRCV, CRV, false, EPIV)              \
  }
  if (d.epi) {
    if (d.src == SRC_LOAD) {
      NS2_NL(SRC_LOAD, false, true)
    } else {
      NS2_NL(SRC_FMG, false, true)
    }
  } else if (d.src == SRC_LOAD) {
    if (d.cr) {
      NS2_NL(SRC_LOAD, true, false)
    } else {
      NS2_NL(SRC_LOAD, false, false)
    }
  } else if (d.src == SRC_CORR) {
    if (d.cr) {
      NS2_NL(SRC_CORR, true, false)
    } else {
      NS2_NL(SRC_CORR, false, false)
    }
  } else {
    if (d.cr) {
      NS2_NL(SRC_FMG, true, false)
    } else {
      NS2_NL(SRC_FMG, false, false)
    }
  }
#undef NS2_NL
#undef NS2_OM
}


}  // namespace fmgsr
