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
#include <type_traits>

#include "fmgsr_chain.cuh"
#include "fmgsr_internal.h"
#include "visit_common.cuh"

namespace fmgsr {

// Lane width (RHS columns per lane).  FMGSR_VISIT_CPL=1 forces one column per
// lane, =2 two columns wherever legal; default: automatic (visit_lanes_auto).
static int visit_cpl_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_VISIT_CPL");
    v = (e && std::string(e) == "1") ? 1 : (e && std::string(e) == "2") ? 2 : 0;
  }
  return v;
}
static bool visit_cpl2_enabled() { return visit_cpl_env() != 1; }

// SM sub-partitions (warp schedulers) of the device the launch runs on
int visit_smsps() {
  static int n = 0;
  if (!n) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    n = 4 * sms;
  }
  return n;
}

// A visit is issue-latency bound when its chains cannot fill the GPU: one lane
// runs one sequential chain, so with at most one warp per SM sub-partition
// every warp issues alone and a pair costs its own instruction count (about
// 2 x 50 fp64 issue cycles per pair with two columns per lane).  One column
// per lane then halves each warp's instructions per pair and doubles the
// number of sub-partitions at work (config-5 P = 16 / 64).  With more chains
// than that, two columns per lane move the same bytes with fewer instructions.
template <typename T>
static bool visit_few_chains(const VisitDesc<T>& d) {
  const i64 P = d.olo ? d.P : (d.p_count >= 0 ? d.p_count : d.n / d.W);
  const i64 warps1 = P * ((d.B + 31) / 32);
  return warps1 <= visit_smsps();
}

// short patches (W <= 16): one warp per group of patches (kernels_group.cu)
template <typename T>
bool try_group_visit(const VisitDesc<T>& d, cudaStream_t s);

// FAS-correction up visits with several patches per warp (kernels_visit_mp.cu)
bool visit_up_mp(const VisitDesc<double>& d, bool r4, cudaStream_t s);

// the fills live in kernels_visit_{d,f,v2d,v2f}.cu (one instantiation each,
// compiled in parallel)
template <typename TV, typename T, int SHAPE, typename TM = TV>
void visit_fill_launch(const VisitDesc<T>& d, cudaStream_t s);

// fp32 fields, fp64 arithmetic (kernels_visit_m{d,v2d}.cu); only T = float
template <typename T>
static void visit_launch_mixed(const VisitDesc<T>& d, bool v2, bool few, cudaStream_t s) {
  (void)d, (void)v2, (void)few, (void)s;
  require(false, "visit: fp64 arithmetic applies to fp32 fields only");
}
template <>
void visit_launch_mixed<float>(const VisitDesc<float>& d, bool v2, bool few, cudaStream_t s) {
  require(((uintptr_t)d.E & 15) == 0 && ((uintptr_t)d.E_out & 15) == 0,
          "visit: fp64 edge records must be 16-byte aligned");
  if (v2) visit_fill_launch<V2<double>, float, SHAPE_WIDE, V2<float>>(d, s);
  else if (few) visit_fill_launch<double, float, SHAPE_DEEP, float>(d, s);
  else visit_fill_launch<double, float, SHAPE_WIDE, float>(d, s);
}

// Two columns per lane: whole 64-column row groups, 2-element-aligned rows
// and pointers, uniform geometry (no explicit patch arrays).  A shard slab's
// edge outbox [2][5][ldE] has the same memory layout with either lane type
// once B % 64 == 0 (ldE = B doubles = 2 x the V2 stride), so the slab-edge
// fix-up and the transfers are unchanged.
// Measured on config 2 (tools/visit_breakdown.py): mid-level visits 10-25 %
// faster, 3.29 -> 3.08 ms per cycle; config 5 fp32 8.66 -> 6.84 ms.
template <typename T>
static bool visit_cpl2_ok(const VisitDesc<T>& d) {
  constexpr uintptr_t A = 2 * sizeof(T);
  auto al = [](const void* p) { return ((uintptr_t)p & (A - 1)) == 0; };
  // fp64 Pi + Kaczmarz (the SR up visit) measured slower with two columns per
  // lane (U_16 of config 2: 270 vs 226 us; 16-byte lanes need ~220 registers
  // there); every other visit kind, and every fp32 visit, is faster
  if ((sizeof(T) == 8 || d.f64_arith) && d.src == SRC_FMG && d.cr) return false;
  if (visit_cpl_env() == 0 && visit_few_chains(d)) return false;
  return visit_cpl2_enabled() && d.B % 64 == 0 && d.ld % 2 == 0 && !d.olo && al(d.u_src) && al(d.uH) && al(d.uc) && al(d.f) &&
         al(d.u_out) && al(d.uH_out) && al(d.fH_out) && al(d.E) && al(d.E_out) && al(d.fun_w) &&
         al(d.fun_part);
}

// R4 launch shape (4-pair ring, 128-register bound: four CTAs per SM) for the
// two-column fp64 down visits (plain load + fused restriction: 160 registers
// and a 64 KB ring hold WIDE to three CTAs per SM) and FAS-correction up
// visits (an 80 KB ring holds WIDE to two), when the launch has more warps
// than one WIDE wave (148 SMs x 12 warps): then the fuller last wave and the
// extra resident warps outweigh the shallower ring.  Measured on config 4
// (4096 warps per visit, tools/visit_breakdown.py): level-17..23 down visits
// 3-7 % and up visits 1-7 % faster; with fewer warps than one wave (config 2,
// 1024) the shallower ring loses (3.029 -> 3.050 ms), and the FMG top visits
// spill at 128 registers, so they stay WIDE.  FMGSR_VISIT_R4 = 0 (never),
// d / du (down / down and up visits regardless of size), all (every
// two-column fp64 visit) for A/B runs.
template <typename T>
static bool visit_r4(const VisitDesc<T>& d) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_VISIT_R4");
    const std::string x = e ? e : "";
    v = x == "0" ? 0 : x == "d" ? 1 : x == "du" ? 2 : x == "all" ? 3 : 4;
  }
  const bool down = d.src == SRC_LOAD && d.epi, up = d.src == SRC_CORR && !d.epi && !d.cr;
  if (v == 0) return false;
  if (v == 3) return true;
  if (v == 1) return down;
  if (v == 2) return down || up;
  const i64 P = d.p_count >= 0 ? d.p_count : d.n / d.W;
  const i64 warps = P * ((d.B / 2 + 31) / 32);
  return (down || up) && warps > 12 * (i64)visit_smsps() / 4;
}

template <typename T>
void launch_visit(const VisitDesc<T>& d, cudaStream_t s) {
  require(d.n >= 2 && is_pow2(d.n), "visit: level size must be a power of two >= 2");
  require(d.B >= 1 && d.ld >= d.B, "visit: need 1 <= B <= ld");
  require(d.f != nullptr, "visit: f is null");
  require(!d.fun_part || (!d.epi && !d.olo && d.p_count < 0 &&
                          ((d.src == SRC_FMG && d.cr) || (d.src == SRC_CORR && !d.cr))),
          "visit: functional output only on a final up visit");
  if (d.olo) {
    require(d.src == SRC_LOAD && !d.epi, "visit: patch arrays only with plain loads");
  } else {
    require(d.W >= 2 && d.W % 2 == 0 && d.n % d.W == 0, "visit: owned width must be even and divide n");
    require(d.b >= 0, "visit: negative buffer");
    if (d.p_count >= 0)
      require(d.p_begin >= 0 && d.p_begin + d.p_count <= d.n / d.W,
              "visit: patch range outside the level");
  }
  require(!(d.left_remote || d.right_remote) || (d.E_out && d.epi), "visit: remote edges need an outbox");
  if (d.src == SRC_LOAD) require(d.u_src != nullptr, "visit: LOAD needs u_src");
  if (d.src == SRC_CORR) require(d.u_src && d.uH, "visit: CORR needs u_src and uH");
  if (d.src == SRC_FMG) require(d.uH && d.n >= 8, "visit: FMG needs uH with >= 4 coarse cells");
  if (d.cr && d.src != SRC_FMG) require(d.uc != nullptr, "visit: CR needs uc");
  if (d.epi) {
    require(d.fH_out && d.E && d.cnt, "visit: epilogue buffers missing");
  } else {
    require(d.u_out != nullptr || d.fun_part != nullptr, "visit: u_out is null");
  }
  if (try_group_visit(d, s)) return;  // short patches (fuses the restriction from W = 2)
  if (d.epi) require(d.W >= 4 && d.n >= 8, "visit: fused restriction needs owned width >= 4");
  if (d.f64_arith) {
    require(!d.fun_part, "visit: no functional output with fp64 arithmetic on fp32 fields");
    visit_launch_mixed(d, visit_cpl2_ok(d), visit_few_chains(d), s);
  } else if (visit_cpl2_ok(d)) {
    bool r4 = false;
    if constexpr (std::is_same<T, double>::value) {
      r4 = visit_r4(d);
      // up visits of launches that overfill the warp slots: several patches per warp
      if (visit_up_mp(d, r4, s)) {
        check_launch("visit_up_mp_kernel");
        return;
      }
      if (r4) visit_fill_launch<V2<T>, T, SHAPE_R4>(d, s);
    }
    if (!r4) visit_fill_launch<V2<T>, T, SHAPE_WIDE>(d, s);
  } else if (visit_few_chains(d)) {
    visit_fill_launch<T, T, SHAPE_DEEP>(d, s);
  } else {
    visit_fill_launch<T, T, SHAPE_WIDE>(d, s);
  }
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
  const T ih = (T)pow4(lv), iH = (T)pow4(lv - 1);
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
