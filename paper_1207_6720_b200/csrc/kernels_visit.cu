// kernels_visit.cu -- the patch-sweep kernels.
//
// visit_kernel: one warp per (patch, 32 RHS), one lane per chain.  Fuses the
// level visit of the FMG cycle (reference cycles.py:187-199, 95-134):
//   prologue  : u_in from LOAD / FAS correction / FMG prolongation (+CR)
//   smoother  : additive patch Gauss-Seidel, ns = 1 (_kernels_numba.py:60-92)
//   epilogue  : owned store, and optionally restriction + tau for the next
//               coarser level (stencils.py:39-47, 108-125) with the patch-
//               boundary coarse cells completed by the second-arriving warp.
// smooth_scratch_kernel: any ns; the extended window is staged per chain in
// a global scratch and replayed exactly as the reference does (Kaczmarz
// pass, GS pass, direction flip per repetition, owned write-back).
#include <cmath>
#include <cstdlib>
#include <string>

#include "fmgsr_chain.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

template <typename T>
struct VisitArgs {
  i64 n, ld, W, b, P, nc, p_begin, qlo, qhi;
  T* E_out;
  bool left_remote, right_remote;
  int B, nrg;
  GsCoef<T> gc;
  KzCoef<T> kz;
  T inv_H2;
  bool write_u;
  const T *u_src, *uH, *uc, *f;
  T *u_out, *uH_out, *fH_out, *E;
  int* cnt;
  const i64 *olo, *ohi, *elo, *ehi;
  const T* fun_w;  // FUNC: weights (nullptr: unit)
  T* fun_part;     // FUNC: per-(patch, column) partial sums [P][nrg * 32]
};

constexpr int VNT = 128;  // threads per block of the visit kernel
constexpr int VD = 8;     // cp.async ring depth (pairs) per lane

template <typename T, int SRC, bool CR>
__host__ __device__ constexpr size_t visit_ring_bytes() {
  return (size_t)VD * SrcRows<SRC, CR>::R * VNT * sizeof(T);
}
template <typename T, int SRC, bool CR>
__host__ __device__ constexpr size_t visit_smem_bytes() {  // staging ring + one mbarrier per (warp, slot)
  return visit_ring_bytes<T, SRC, CR>() + (size_t)(VNT / 32) * VD * 8;
}

template <typename T, int SRC, bool CR, bool EPI, bool OMEGA1, bool BULK, bool FUNC>
__global__ void __launch_bounds__(VNT, 4) visit_kernel(const VisitArgs<T> a) {
  extern __shared__ __align__(128) unsigned char visit_smem[];
  const int lane = threadIdx.x & 31;
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 pl = gw / a.nrg;  // patch index within the launched range
  const int rg = (int)(gw - pl * a.nrg);
  if (pl >= a.P) return;  // warp-uniform
  const i64 p = a.p_begin + pl;
  const int r = rg * 32 + lane;
  const bool store = r < a.B;
  const int rr = store ? r : a.B - 1;

  i64 os, oe, ws, we;
  if (a.olo) {
    os = a.olo[p];
    oe = a.ohi[p];
    ws = a.elo[p];
    we = a.ehi[p];
  } else {
    os = p * a.W;
    oe = os + a.W;
    ws = os - a.b > 0 ? os - a.b : 0;
    we = oe + a.b < a.n ? oe + a.b : a.n;
  }

  Chain<T, SRC, CR, EPI, OMEGA1, VNT, VD, BULK, FUNC> ch;
  ch.lane = lane;
  ch.bars = reinterpret_cast<unsigned long long*>(visit_smem + visit_ring_bytes<T, SRC, CR>()) +
            (threadIdx.x >> 5) * VD;
  if (BULK) {
    if (lane == 0)
      for (int k = 0; k < VD; k++) mbar_init(ch.bars + k, 1);
    mbar_fence_init();
    __syncwarp();
  }
  ch.src.u = a.u_src ? a.u_src + rr : nullptr;
  ch.src.uH = a.uH ? a.uH + rr : nullptr;
  ch.src.uc = a.uc ? a.uc + rr : nullptr;
  ch.src.f = a.f + rr;
  ch.src.ld = a.ld;
  ch.src.nc = a.nc;
  ch.src.kz = a.kz;
  ch.src.wlo = ws >> 1;
  ch.src.whi = we >> 1;
  ch.src.qlo = a.qlo;
  ch.src.qhi = a.qhi;
  ch.gc = a.gc;
  ch.n = a.n;
  ch.nc = a.nc;
  ch.ld = a.ld;
  ch.ws = ws;
  ch.os = os;
  ch.oe = oe;
  ch.store = store;
  ch.ring = reinterpret_cast<T*>(visit_smem) + threadIdx.x;
  ch.out = (a.u_out && (!EPI || a.write_u)) ? a.u_out + r : nullptr;
  ch.fw = (FUNC && a.fun_w) ? a.fun_w + rr : nullptr;
  ch.facc = T(0);
  if (!EPI) {
    ch.epi = nullptr;
    ch.run(we);
    if (FUNC) a.fun_part[p * ((i64)a.nrg * 32) + r] = ch.facc;
    return;
  }
  Epilogue<T> ep;
  ep.inv_h2 = a.gc.inv_h2;
  ep.inv_H2 = a.inv_H2;
  ep.left_dom = (os == 0);
  ep.right_dom = (oe == a.n);
  ep.write_uH = a.uH_out != nullptr;
  ep.uH_out = a.uH_out ? a.uH_out + r : nullptr;
  ep.fH_out = a.fH_out + r;
  ep.ld = a.ld;
  ep.nc = a.nc;
  ep.cnt = 0;
  ep.up2 = ep.up1 = ep.Lprev = ep.Rm2 = ep.Rm1 = ep.Rfm1 = T(0);
  ch.epi = &ep;
  ch.run(we);
  EdgeRec<T> right;
  ep.finish(store, right);
  const i64 ldE = (i64)a.nrg * 32;
  if (!ep.left_dom) {
    if (pl == 0 && a.left_remote) {  // slab edge: the neighbour shard finishes it
#pragma unroll
      for (int k = 0; k < 5; k++) a.E_out[(0 * 5 + k) * ldE + r] = ep.left.v[k];
    } else {
      edge_arrive(a.E, a.cnt, ldE, a.nrg, p, 1, ep.left, lane, rg, r, store, ep.fH_out, a.ld, os,
                  ep.inv_h2, ep.inv_H2);
    }
  }
  if (!ep.right_dom) {
    if (pl == a.P - 1 && a.right_remote) {
#pragma unroll
      for (int k = 0; k < 5; k++) a.E_out[(1 * 5 + k) * ldE + r] = right.v[k];
    } else {
      edge_arrive(a.E, a.cnt, ldE, a.nrg, p + 1, 0, right, lane, rg, r, store, ep.fH_out, a.ld, oe,
                  ep.inv_h2, ep.inv_H2);
    }
  }
}

template <typename T>
static GsCoef<T> make_coef(i64 n, double omega) {
  int k = level_of(n);
  GsCoef<T> g;
  double inv_h2 = (double)((i64)1 << (2 * k));
  g.inv_h2 = (T)inv_h2;
  g.rdiag = (T)(1.0 / (2.0 * inv_h2));  // exact power of two
  g.diag_b = (T)(3.0 * inv_h2);
  g.omega = (T)omega;
  g.diag_i = (T)(2.0 * inv_h2);
  return g;
}

// FMGSR_VISIT_STAGING=cpasync forces the per-lane cp.async staging (A/B tests)
static bool visit_bulk_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_VISIT_STAGING");
    v = (e && std::string(e) == "cpasync") ? 0 : 1;
  }
  return v == 1;
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

template <typename T, int SRC, bool CR, bool EPI, bool OMEGA1, bool BULK, bool FUNC = false>
static void launch_visit_k(const VisitArgs<T>& a, i64 blocks, cudaStream_t s) {
  constexpr size_t smem = visit_smem_bytes<T, SRC, CR>();
  auto k = visit_kernel<T, SRC, CR, EPI, OMEGA1, BULK, FUNC>;
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
    attr = true;
  }
  k<<<(unsigned)blocks, VNT, smem, s>>>(a);
}

// Bulk (TMA) staging needs whole 32-column row segments at 16-byte alignment.
template <typename T>
static bool bulk_ok(const VisitArgs<T>& a) {
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  return a.B % 32 == 0 && (a.ld * sizeof(T)) % 16 == 0 && al(a.f) &&
         (!a.u_src || al(a.u_src)) && (!a.uH || al(a.uH)) && (!a.uc || al(a.uc)) &&
         visit_bulk_enabled();
}

template <typename T, int SRC, bool CR, bool EPI>
static void launch_visit_t(const VisitArgs<T>& a, cudaStream_t s) {
  i64 warps = a.P * a.nrg;
  i64 blocks = (warps + VNT / 32 - 1) / (VNT / 32);
  const bool om1 = a.gc.omega == T(1);
  // bulk (TMA) staging pays off where per-lane LDGSTS saturates the MIO
  // queue: sources with >= 5 staged rows per pair (the FAS-correction visits);
  // measured slower than cp.async for 3-4 rows (profiles/r01 notes)
  const bool bulk = SrcRows<SRC, CR>::R >= 5 && bulk_ok(a);
  // functional output of the final up visit (non-SR: FAS correction; SR: Pi + CR)
  if constexpr (!EPI && ((SRC == SRC_FMG && CR) || (SRC == SRC_CORR && !CR))) {
    if (a.fun_part) {
      if (om1) {
        if (bulk) launch_visit_k<T, SRC, CR, EPI, true, true, true>(a, blocks, s);
        else launch_visit_k<T, SRC, CR, EPI, true, false, true>(a, blocks, s);
      } else {
        if (bulk) launch_visit_k<T, SRC, CR, EPI, false, true, true>(a, blocks, s);
        else launch_visit_k<T, SRC, CR, EPI, false, false, true>(a, blocks, s);
      }
      return;
    }
  }
  if (om1) {
    if (bulk) launch_visit_k<T, SRC, CR, EPI, true, true>(a, blocks, s);
    else launch_visit_k<T, SRC, CR, EPI, true, false>(a, blocks, s);
  } else {
    if (bulk) launch_visit_k<T, SRC, CR, EPI, false, true>(a, blocks, s);
    else launch_visit_k<T, SRC, CR, EPI, false, false>(a, blocks, s);
  }
}

template <typename T>
void launch_visit(const VisitDesc<T>& d, cudaStream_t s) {
  require(d.n >= 2 && is_pow2(d.n), "visit: level size must be a power of two >= 2");
  require(d.B >= 1 && d.ld >= d.B, "visit: need 1 <= B <= ld");
  require(d.f != nullptr, "visit: f is null");
  VisitArgs<T> a;
  a.n = d.n;
  a.ld = d.ld;
  a.B = d.B;
  a.nrg = (d.B + 31) / 32;
  a.nc = d.n / 2;
  a.gc = make_coef<T>(d.n, d.omega);
  a.inv_H2 = (T)(double)((i64)1 << (2 * (level_of(d.n) - 1)));
  a.kz = make_kz<T>(d.proj_diag);
  a.write_u = d.write_u;
  a.u_src = d.u_src;
  a.uH = d.uH;
  a.uc = d.uc;
  a.f = d.f;
  a.u_out = d.u_out;
  a.uH_out = d.uH_out;
  a.fH_out = d.fH_out;
  a.E = d.E;
  a.cnt = d.cnt;
  a.olo = d.olo;
  a.ohi = d.ohi;
  a.elo = d.elo;
  a.ehi = d.ehi;
  a.p_begin = 0;
  a.qlo = d.qlo >= 0 ? d.qlo : 0;
  a.qhi = d.qhi >= 0 ? d.qhi : a.nc - 1;
  a.E_out = d.E_out;
  a.left_remote = d.left_remote;
  a.right_remote = d.right_remote;
  a.fun_w = d.fun_w;
  a.fun_part = d.fun_part;
  require(!d.fun_part || (!d.epi && !d.olo && d.p_count < 0 &&
                          ((d.src == SRC_FMG && d.cr) || (d.src == SRC_CORR && !d.cr))),
          "visit: functional output only on a final up visit");
  if (d.olo) {
    require(d.src == SRC_LOAD && !d.epi, "visit: patch arrays only with plain loads");
    a.P = d.P;
    a.W = 0;
    a.b = 0;
  } else {
    require(d.W >= 2 && d.W % 2 == 0 && d.n % d.W == 0, "visit: owned width must be even and divide n");
    require(d.b >= 0, "visit: negative buffer");
    a.W = d.W;
    a.b = d.b;
    a.P = d.n / d.W;
    if (d.p_count >= 0) {
      require(d.p_begin >= 0 && d.p_begin + d.p_count <= a.P, "visit: patch range outside the level");
      a.p_begin = d.p_begin;
      a.P = d.p_count;
    }
  }
  require(!(d.left_remote || d.right_remote) || (d.E_out && d.epi), "visit: remote edges need an outbox");
  if (d.src == SRC_LOAD) require(d.u_src != nullptr, "visit: LOAD needs u_src");
  if (d.src == SRC_CORR) require(d.u_src && d.uH, "visit: CORR needs u_src and uH");
  if (d.src == SRC_FMG) require(d.uH && d.n >= 8, "visit: FMG needs uH with >= 4 coarse cells");
  if (d.cr && d.src != SRC_FMG) require(d.uc != nullptr, "visit: CR needs uc");
  if (d.epi) {
    require(d.W >= 4 && d.n >= 8, "visit: fused restriction needs owned width >= 4");
    require(d.fH_out && d.E && d.cnt, "visit: epilogue buffers missing");
  } else {
    require(d.u_out != nullptr || d.fun_part != nullptr, "visit: u_out is null");
  }
  if (a.P == 0) return;
#define FMGSR_DISPATCH(SRCV)                                                    \
  if (d.cr) {                                                                  \
    if (d.epi) launch_visit_t<T, SRCV, true, true>(a, s);                      \
    else launch_visit_t<T, SRCV, true, false>(a, s);                           \
  } else {                                                                     \
    if (d.epi) launch_visit_t<T, SRCV, false, true>(a, s);                     \
    else launch_visit_t<T, SRCV, false, false>(a, s);                          \
  }
  if (d.src == SRC_LOAD) {
    FMGSR_DISPATCH(SRC_LOAD)
  } else if (d.src == SRC_CORR) {
    FMGSR_DISPATCH(SRC_CORR)
  } else {
    FMGSR_DISPATCH(SRC_FMG)
  }
#undef FMGSR_DISPATCH
  check_launch("visit_kernel");
}

// ---------------------------------------------------------------------------
// Any-ns smoother with a staged window (reference _kernels_numba.py:60-92 in
// its literal form).  Scratch layout: [row][sld], one column per chain lane,
// patch p owning rows soff(p) .. soff(p) + (hi - lo).
// ---------------------------------------------------------------------------
template <typename T>
struct ScratchArgs {
  i64 n, ld, W, b, P, ns, sld;
  int B, nrg;
  GsCoef<T> gc;
  KzCoef<T> kz;
  const i64 *olo, *ohi, *elo, *ehi, *soff;
  const T *u_in, *f, *uc;
  T *out, *scratch;
};

template <typename T, bool CR, bool NL>
__global__ void __launch_bounds__(128) smooth_scratch_kernel(const ScratchArgs<T> a) {
  const int lane = threadIdx.x & 31;
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 p = gw / a.nrg;
  const int rg = (int)(gw - p * a.nrg);
  if (p >= a.P) return;
  const int r = rg * 32 + lane;
  const bool store = r < a.B;
  const int rr = store ? r : a.B - 1;
  i64 os, oe, ws, we, off;
  if (a.olo) {
    os = a.olo[p];
    oe = a.ohi[p];
    ws = a.elo[p];
    we = a.ehi[p];
    off = a.soff[p];
  } else {
    os = p * a.W;
    oe = os + a.W;
    ws = os - a.b > 0 ? os - a.b : 0;
    we = oe + a.b < a.n ? oe + a.b : a.n;
    off = p * (a.W + 2 * a.b + 2);
  }
  const i64 n = a.n, ld = a.ld;
  const i64 lo = ws > 0 ? ws - 1 : 0;
  const i64 hi = we < n ? we + 1 : n;
  T* S0 = a.scratch + off * a.sld + r;  // window cell i lives at S0[(i - lo) * sld]
  const i64 sld = a.sld;
#define S(i) S0[((i) - lo) * sld]
  const T* f = a.f + rr;
  const T* ui = a.u_in + rr;
  for (i64 i = lo; i < hi; i++) S(i) = ldg(ui + i * ld);
  bool forward = true;
  for (i64 rep = 0; rep < a.ns; rep++) {
    if (CR) {
      const T* uc = a.uc + rr;
      for (i64 j = ws >> 1; j < (we >> 1); j++) {
        T x = S(2 * j), y = S(2 * j + 1);
        kaczmarz_pair(x, y, ldg(uc + j * ld), a.kz);
        S(2 * j) = x;
        S(2 * j + 1) = y;
      }
    }
    if (forward) {
      T uL = ws > 0 ? S(ws - 1) : T(0);
      T cur = S(ws);
      for (i64 i = ws; i < we; i++) {
        T nxt = (i + 1 < hi) ? S(i + 1) : T(0);
        T v = NL ? gs_cell_nl(a.gc, i, n, uL, cur, nxt, ldg(f + i * ld))
                 : gs_cell(a.gc, i, n, uL, cur, nxt, ldg(f + i * ld));
        S(i) = v;
        uL = v;
        cur = nxt;
      }
    } else {
      T uR = we < n ? S(we) : T(0);
      T cur = S(we - 1);
      for (i64 i = we - 1; i >= ws; i--) {
        T prv = (i - 1 >= lo) ? S(i - 1) : T(0);
        T v = NL ? gs_cell_nl(a.gc, i, n, prv, cur, uR, ldg(f + i * ld))
                 : gs_cell(a.gc, i, n, prv, cur, uR, ldg(f + i * ld));
        S(i) = v;
        uR = v;
        cur = prv;
      }
    }
    forward = !forward;
  }
  if (store) {
    T* o = a.out + r;
    for (i64 i = os; i < oe; i++) o[i * ld] = S(i);
  }
#undef S
}

template <typename T>
void launch_smooth_scratch(const ScratchDesc<T>& d, cudaStream_t s) {
  require(d.n >= 2 && is_pow2(d.n), "smooth: level size must be a power of two >= 2");
  require(d.B >= 1 && d.ld >= d.B, "smooth: need 1 <= B <= ld");
  require(d.ns >= 1, "smooth: ns must be >= 1");
  require(d.u_in && d.f && d.out && d.scratch, "smooth: null pointer");
  ScratchArgs<T> a;
  a.n = d.n;
  a.ld = d.ld;
  a.B = d.B;
  a.nrg = (d.B + 31) / 32;
  require(d.sld >= (i64)a.nrg * 32, "smooth: scratch stride too small");
  a.sld = d.sld;
  a.ns = d.ns;
  a.gc = make_coef<T>(d.n, d.omega);
  a.kz = make_kz<T>(d.proj_diag);
  a.olo = d.olo;
  a.ohi = d.ohi;
  a.elo = d.elo;
  a.ehi = d.ehi;
  a.soff = d.soff;
  a.u_in = d.u_in;
  a.f = d.f;
  a.uc = d.uc;
  a.out = d.out;
  a.scratch = d.scratch;
  if (d.olo) {
    require(d.soff != nullptr, "smooth: patch arrays need scratch offsets");
    a.P = d.P;
    a.W = a.b = 0;
  } else {
    require(d.W >= 1 && d.n % d.W == 0, "smooth: owned width must divide n");
    a.W = d.W;
    a.b = d.b;
    a.P = d.n / d.W;
  }
  if (a.P == 0) return;
  i64 blocks = (a.P * a.nrg + 3) / 4;
  if (d.nonlinear) {
    if (d.uc) smooth_scratch_kernel<T, true, true><<<(unsigned)blocks, 128, 0, s>>>(a);
    else smooth_scratch_kernel<T, false, true><<<(unsigned)blocks, 128, 0, s>>>(a);
  } else {
    if (d.uc) smooth_scratch_kernel<T, true, false><<<(unsigned)blocks, 128, 0, s>>>(a);
    else smooth_scratch_kernel<T, false, false><<<(unsigned)blocks, 128, 0, s>>>(a);
  }
  check_launch("smooth_scratch_kernel");
}

// Slab-boundary coarse cell (which = 0: s/2 - 1, owned by the left shard;
// which = 1: s/2, owned by the right shard) from the two edge records.
template <typename T>
__global__ void k_edge_fix(const T* __restrict__ L, const T* __restrict__ R, T* fH, i64 s, i64 nf,
                           i64 ld, int B, i64 ldE, int which) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const int lv = level_of(nf);
  const T ih = (T)(double)((i64)1 << (2 * lv)), iH = (T)(double)((i64)1 << (2 * (lv - 1)));
  T Lr[5], Rr[5];
#pragma unroll
  for (int k = 0; k < 5; k++) {
    Lr[k] = L[k * ldE + r];
    Rr[k] = R[k * ldE + r];
  }
  T fL, fR;
  edge_finish(Lr, Rr, ih, iH, fL, fR);
  if (which != 1) fH[(s / 2 - 1) * ld + r] = fL;  // 0: left cell, 1: right cell, 2: both
  if (which != 0) fH[(s / 2) * ld + r] = fR;
}

// Functional of a stored field with the fused visit's summation order: per
// (patch, column) a sequential sum of w_i u_i over the owned cells, then
// (k_functional_reduce) a sequential sum over patches, times `scale`.
template <typename T>
__global__ void k_functional_field(const T* __restrict__ u, const T* __restrict__ w, i64 n, i64 W,
                                   i64 ld, int B, T* part, i64 ldp) {
  const i64 k = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 P = n / W;
  if (k >= P * ldp) return;
  const i64 p = k / ldp;
  const int r = (int)(k - p * ldp);
  const int rr = r < B ? r : B - 1;
  T acc = T(0);
  for (i64 i = p * W; i < (p + 1) * W; i++)
    acc = xadd(acc, w ? xmul(w[i * ld + rr], u[i * ld + rr]) : u[i * ld + rr]);
  part[p * ldp + r] = acc;
}
template <typename T>
__global__ void k_functional_reduce(const T* __restrict__ part, i64 P, i64 ldp, int B, T scale,
                                    T* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  T acc = T(0);
  for (i64 p = 0; p < P; p++) acc = xadd(acc, part[p * ldp + r]);
  out[r] = xmul(acc, scale);
}
template <typename T>
void launch_functional_field(const T* u, const T* w, i64 n, i64 W, i64 ld, int B, T* part,
                             cudaStream_t s) {
  const i64 ldp = ((B + 31) / 32) * 32, items = (n / W) * ldp;
  k_functional_field<T><<<(unsigned)((items + 255) / 256), 256, 0, s>>>(u, w, n, W, ld, B, part, ldp);
  check_launch("functional_field");
}
template <typename T>
void launch_functional_reduce(const T* part, i64 P, int B, T scale, T* out, cudaStream_t s) {
  const i64 ldp = ((B + 31) / 32) * 32;
  k_functional_reduce<T><<<(B + 127) / 128, 128, 0, s>>>(part, P, ldp, B, scale, out);
  check_launch("functional_reduce");
}
template void launch_functional_field<double>(const double*, const double*, i64, i64, i64, int, double*, cudaStream_t);
template void launch_functional_field<float>(const float*, const float*, i64, i64, i64, int, float*, cudaStream_t);
template void launch_functional_reduce<double>(const double*, i64, int, double, double*, cudaStream_t);
template void launch_functional_reduce<float>(const float*, i64, int, float, float*, cudaStream_t);

template <typename T>
void launch_edge_fix(const T* rec_left, const T* rec_right, T* fH, i64 s, i64 nf, i64 ld, int B,
                     int which, cudaStream_t st) {
  const i64 ldE = ((B + 31) / 32) * 32;
  k_edge_fix<T><<<(B + 127) / 128, 128, 0, st>>>(rec_left, rec_right, fH, s, nf, ld, B, ldE, which);
  check_launch("edge_fix");
}
template void launch_edge_fix<double>(const double*, const double*, double*, i64, i64, i64, int, int, cudaStream_t);
template void launch_edge_fix<float>(const float*, const float*, float*, i64, i64, i64, int, int, cudaStream_t);

template void launch_visit<double>(const VisitDesc<double>&, cudaStream_t);
template void launch_visit<float>(const VisitDesc<float>&, cudaStream_t);
template void launch_smooth_scratch<double>(const ScratchDesc<double>&, cudaStream_t);
template void launch_smooth_scratch<float>(const ScratchDesc<float>&, cudaStream_t);

}  // namespace fmgsr
