// kernels_ns2.cu -- the V(2,2) patch smoother (ns = 2) as two streaming chains.
//
// Reference semantics (_kernels_numba.py:79-91 with ns = 2): per patch, on a
// private copy of the window [ws-1, we+1): Kaczmarz pass + forward GS over
// [ws, we), then Kaczmarz pass + backward GS, owned cells written back.  The
// backward sweep starts at the right end of the forward-swept window, so the
// window must be kept between the sweeps: each lane spills its forward sweep
// to a private scratch column ([row][chain], coalesced per warp) and streams
// it back in reverse.
//   forward : the visit prologue (plain / FAS correction / FMG prolongation),
//             first Kaczmarz pass just in time, GS forward (linear or the
//             Newton step of the nonlinear path); every window cell -> scratch
//   backward: second Kaczmarz pass just in time on the scratch values (pair
//             j is projected when the sweep reaches it, before either cell is
//             updated), GS backward, owned cells -> u_out.
// Both chains stage their rows D-1 pairs ahead by per-lane cp.async.
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
  const T *u_src, *uH, *uc, *f;
  T *u_out, *scratch;
};

__device__ __forceinline__ i64 imax(i64 a, i64 b) { return a > b ? a : b; }
__device__ __forceinline__ i64 imin(i64 a, i64 b) { return a < b ? a : b; }

template <typename T, int SRC, bool CR, bool NL, bool OMEGA1>
__global__ void __launch_bounds__(NT2, 4) ns2_kernel(const Ns2Args<T> a) {
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
    T* sp = Sc + (2 * q - lo) * sld;
    for (; q <= qf_hi; q++) {
      cp_wait<D2 - 2>();
      Raw<T> rw = src.template fetch<NT2>(slot(q + 1));
      src.template issue<NT2>(slot(q), q + D2);
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
    }
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
  T* out = a.u_out + r;
  auto bwd_slow = [&](i64 j) {
    const i64 i1 = 2 * j + 1, i0 = 2 * j;
    T b0 = T(0), b1 = T(0), h0 = T(0), h1 = T(0);
    if (j - 1 >= jb) pair_vals(j - 1, b0, b1, h0, h1);
    if (i1 >= ws && i1 < we) {
      const T v = gs2<T, NL>(gc, i1, n, a0, a1, uR, g1);
      if (store && i1 >= os && i1 < oe) out[i1 * ld] = v;
      uR = v;
    }
    // cell 2j: its left neighbour 2j-1 is the second cell of pair j-1
    if (i0 >= ws && i0 < we) {
      const T v = gs2<T, NL>(gc, i0, n, b1, a0, uR, g0);
      if (store && i0 >= os && i0 < oe) out[i0 * ld] = v;
      uR = v;
    }
    a0 = b0;
    a1 = b1;
    g0 = h0;
    g1 = h1;
  };
  // fast pairs: both cells owned interior cells, pair j-1 exists
  const i64 jf_hi = (imin(oe - 1, n - 2) - 1) >> 1;
  const i64 jf_lo = imax((imax(os, 1) + 1) >> 1, jb + 1);
  i64 j = jt;
  for (; j >= jb && j > jf_hi; j--) bwd_slow(j);
  {
    T* op = out + (2 * j) * ld;
    for (; j >= jf_lo; j--) {
      T b0, b1, h0, h1;
      pair_vals(j - 1, b0, b1, h0, h1);
      const T x1 = gs2i<T, NL, OMEGA1>(gc, a0, a1, uR, g1);
      const T x0 = gs2i<T, NL, OMEGA1>(gc, b1, a0, x1, g0);
      if (store) {
        op[ld] = x1;
        op[0] = x0;
      }
      op -= 2 * ld;
      uR = x0;
      a0 = b0;
      a1 = b1;
      g0 = h0;
      g1 = h1;
    }
  }
  for (; j >= jb; j--) bwd_slow(j);
  cp_wait<0>();
}

}  // namespace

template <typename T>
void launch_smooth_ns2(const Ns2Desc<T>& d, cudaStream_t s) {
  require(d.n >= 8 && is_pow2(d.n), "ns2: level size must be a power of two >= 8");
  require(d.W >= 2 && d.W % 2 == 0 && d.n % d.W == 0, "ns2: owned width must be even and divide n");
  require(d.u_out && d.f && d.scratch, "ns2: null pointer");
  Ns2Args<T> a;
  a.n = d.n;
  a.ld = d.ld;
  a.B = d.B;
  a.nrg = (d.B + 31) / 32;
  a.W = d.W;
  a.b = d.b;
  a.nc = d.n / 2;
  a.P = d.n / d.W;
  a.p_begin = 0;
  a.srows = d.W + 2 * d.b + 2;
  a.sld = (i64)a.nrg * 32;
  require(d.sld >= a.sld, "ns2: scratch stride too small");
  a.sld = d.sld;
  int k = level_of(d.n);
  double ih = (double)((i64)1 << (2 * k));
  a.gc.inv_h2 = (T)ih;
  a.gc.rdiag = (T)(1.0 / (2.0 * ih));
  a.gc.diag_b = (T)(3.0 * ih);
  a.gc.omega = (T)d.omega;
  a.gc.diag_i = (T)(2.0 * ih);
  a.kz.proj_diag = (T)d.proj_diag;
  int e;
  a.kz.pow2 = std::frexp(d.proj_diag, &e) == 0.5;
  a.kz.recip = (T)(a.kz.pow2 ? std::ldexp(1.0, 1 - e) : 1.0 / d.proj_diag);
  a.u_src = d.u_src;
  a.uH = d.uH;
  a.uc = d.uc;
  a.f = d.f;
  a.u_out = d.u_out;
  a.scratch = d.scratch;
  if (d.src == SRC_LOAD) require(d.u_src != nullptr, "ns2: LOAD needs u_src");
  if (d.src == SRC_CORR) require(d.u_src && d.uH, "ns2: CORR needs u_src and uH");
  if (d.src == SRC_FMG) require(d.uH != nullptr, "ns2: FMG needs uH");
  if (d.cr && d.src != SRC_FMG) require(d.uc != nullptr, "ns2: CR needs uc");
  const i64 blocks = (a.P * a.nrg + NT2 / 32 - 1) / (NT2 / 32);
  const size_t smem = (size_t)D2 * 6 * NT2 * sizeof(T);
  const bool om1 = d.omega == 1.0;  // max(R, R2) rows per slot
#define NS2_LAUNCH(SRCV, CRV, NLV)                                                       \
  {                                                                                      \
    auto kf = om1 ? ns2_kernel<T, SRCV, CRV, NLV, true> : ns2_kernel<T, SRCV, CRV, NLV, false>;                                           \
    static bool attr = false;                                                            \
    if (!attr && smem > 48 * 1024) {                                                     \
      check_cuda(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                      (int)smem),                                        \
                 "ns2 smem");                                                            \
      attr = true;                                                                       \
    }                                                                                    \
    kf<<<(unsigned)blocks, NT2, smem, s>>>(a);                                           \
  }
#define NS2_NL(SRCV, CRV)                   \
  if (d.nonlinear) NS2_LAUNCH(SRCV, CRV, true) \
  else NS2_LAUNCH(SRCV, CRV, false)
#define NS2_CR(SRCV)                \
  if (d.cr) {                       \
    NS2_NL(SRCV, true)              \
  } else {                          \
    NS2_NL(SRCV, false)             \
  }
  if (d.src == SRC_LOAD) {
    NS2_CR(SRC_LOAD)
  } else if (d.src == SRC_CORR) {
    NS2_CR(SRC_CORR)
  } else {
    NS2_CR(SRC_FMG)
  }
#undef NS2_CR
#undef NS2_NL
#undef NS2_LAUNCH
  check_launch("ns2_kernel");
}

template void launch_smooth_ns2<double>(const Ns2Desc<double>&, cudaStream_t);
template void launch_smooth_ns2<float>(const Ns2Desc<float>&, cudaStream_t);

}  // namespace fmgsr
