// visit_impl.cuh -- the fused level-visit kernel (visit_kernel) and its
// launch plumbing, instantiated per lane type in kernels_visit_{d,f,v2d,v2f}.cu
// (see kernels_visit.cu for the dispatch and the design notes).
#pragma once

#include <cstdlib>
#include <string>
#include <type_traits>

#include "fmgsr_chain.cuh"
#include "fmgsr_internal.h"
#include "visit_common.cuh"

namespace fmgsr {

// T: the lane's arithmetic type; M: the fields' storage type (T, or fp32
// under fp64 arithmetic).  Edge records and functional partials stay in T.
template <typename T, typename M = T>
struct VisitArgs {
  i64 n, ld, W, b, P, nc, p_begin, qlo, qhi;
  T* E_out;
  bool left_remote, right_remote;
  int B, nrg;
  GsCoef<T> gc;
  KzCoef<T> kz;
  T inv_H2;
  bool write_u;
  const M *u_src, *uH, *uc, *f;
  M *u_out, *uH_out, *fH_out;
  T* E;
  int* cnt;
  const i64 *olo, *ohi, *elo, *ehi;
  const M* fun_w;  // FUNC: weights (nullptr: unit)
  T* fun_part;     // FUNC: per-(patch, column) partial sums [P][nrg * 32]
};

// Launch shapes of the visit kernel (threads per CTA, cp.async ring depth in
// pairs per lane).  WIDE: 8-pair ring -- many chains per SM (the large levels
// at B >= 64), where other warps hide each lane's memory latency.  DEEP:
// 16-pair ring -- few chains (at most one warp per SM sub-partition, scalar
// lanes: config-5 P = 16 / 64): a warp issues alone, so its own ring must
// cover the DRAM latency while the fast loop fetches two pairs ahead.
// R4: 4-pair ring and a 128-register bound -- four CTAs per SM for the visits
// whose 8-pair ring and register count hold them to two or three (A/B:
// FMGSR_VISIT_R4)
template <int SHAPE>
struct VisitShape {
  static constexpr int NT = 128;
  static constexpr int D = SHAPE == SHAPE_WIDE ? 8 : SHAPE == SHAPE_DEEP ? 16 : 4;
};

template <typename M, int SRC, bool CR, int NT, int D>
__host__ __device__ constexpr size_t visit_ring_bytes() {  // the ring holds stored (M) rows
  return (size_t)D * SrcRows<SRC, CR>::R * NT * sizeof(M);
}
template <typename M, int SRC, bool CR, int NT, int D>
__host__ __device__ constexpr size_t visit_smem_bytes() {  // staging ring + one mbarrier per (warp, slot)
  return visit_ring_bytes<M, SRC, CR, NT, D>() + (size_t)(NT / 32) * D * 8;
}

template <typename T, int SRC, bool CR, bool EPI, bool OMEGA1, bool BULK, bool FUNC, int NT, int D,
          typename M = T>
__global__ void __launch_bounds__(NT, (D <= 4 ? 512 : (sizeof(T) > 8 ? 256 : 512)) / NT)
    visit_kernel(const VisitArgs<T, M> a) {
  extern __shared__ __align__(128) unsigned char visit_smem[];
  const int lane = threadIdx.x & 31;
  // 32-bit index math (a launch has < 2^32 threads): no 64-bit division at entry
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nrg = (unsigned)a.nrg;
  const unsigned pl32 = nrg == 1 ? gw : gw / nrg;
  const int rg = (int)(gw - pl32 * nrg);
  const i64 pl = pl32;  // patch index within the launched range
  if (pl >= a.P) return;  // warp-uniform
  const i64 p = a.p_begin + pl;
  const int r = rg * 32 + lane;
  // Lanes past the last RHS column run column B-1's chain (rr) and write its
  // bit-identical values to column B-1, so every store is unconditional and
  // the chain's fast loop has no per-lane branches.
  const bool store = true;
  const int rr = r < a.B ? r : a.B - 1;

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

  Chain<T, SRC, CR, EPI, OMEGA1, NT, D, BULK, FUNC, M> ch;
  ch.lane = lane;
  ch.bars = reinterpret_cast<unsigned long long*>(visit_smem + visit_ring_bytes<M, SRC, CR, NT, D>()) +
            (threadIdx.x >> 5) * D;
  if (BULK) {
    if (lane == 0)
      for (int k = 0; k < D; k++) mbar_init(ch.bars + k, 1);
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
  ch.ring = reinterpret_cast<M*>(visit_smem) + threadIdx.x;
  ch.out = (a.u_out && (!EPI || a.write_u)) ? a.u_out + rr : nullptr;
  ch.fw = (FUNC && a.fun_w) ? a.fun_w + rr : nullptr;
  ch.facc = T(0);
  if (!EPI) {
    ch.epi = nullptr;
    ch.run(we);
    if (FUNC) a.fun_part[p * ((i64)a.nrg * 32) + r] = ch.facc;
    return;
  }
  Epilogue<T, M> ep;
  ep.inv_h2 = a.gc.inv_h2;
  ep.inv_H2 = a.inv_H2;
  ep.left_dom = (os == 0);
  ep.right_dom = (oe == a.n);
  ep.write_uH = a.uH_out != nullptr;
  ep.uH_out = a.uH_out ? a.uH_out + rr : nullptr;
  ep.fH_out = a.fH_out + rr;
  ep.ld = a.ld;
  ep.nc = a.nc;
  ep.cnt = 0;
  ep.up2 = ep.up1 = ep.Lprev = ep.Rm2 = ep.Rm1 = ep.Rfm1 = T(0);
  ch.epi = &ep;
  ch.run(we);
  EdgeRec<T> right;
  ep.finish(store, right);
  const i64 ldE = (i64)a.nrg * 32;
  // slab edges of a shard go to the outbox (the neighbour shard finishes them)
  const bool remL = !ep.left_dom && pl == 0 && a.left_remote;
  const bool remR = !ep.right_dom && pl == a.P - 1 && a.right_remote;
  if (remL) {
#pragma unroll
    for (int k = 0; k < 5; k++) a.E_out[(0 * 5 + k) * ldE + r] = ep.left.v[k];
  }
  if (remR) {
#pragma unroll
    for (int k = 0; k < 5; k++) a.E_out[(1 * 5 + k) * ldE + r] = right.v[k];
  }
  edge_arrive2<T, false, M>(a.E, a.cnt, ldE, a.nrg, lane, rg, r, store, ep.fH_out, a.ld, ep.inv_h2, ep.inv_H2,
               !ep.left_dom && !remL, p, ep.left, os, !ep.right_dom && !remR, p + 1, right, oe);
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


template <typename T, typename M, int SHAPE, int SRC, bool CR, bool EPI, bool OMEGA1, bool BULK,
          bool FUNC = false>
static void launch_visit_k(const VisitArgs<T, M>& a, cudaStream_t s) {
  constexpr int NT = VisitShape<SHAPE>::NT, D = VisitShape<SHAPE>::D;
  constexpr size_t smem = visit_smem_bytes<M, SRC, CR, NT, D>();
  auto k = visit_kernel<T, SRC, CR, EPI, OMEGA1, BULK, FUNC, NT, D, M>;
  if (smem > 48 * 1024)
    require(smem <= (size_t)smem_optin((const void*)k), "visit: shared memory budget exceeded");
  const i64 warps = a.P * a.nrg;
  const i64 blocks = (warps + NT / 32 - 1) / (NT / 32);
  k<<<(unsigned)blocks, NT, smem, s>>>(a);
}

// Bulk (TMA) staging needs whole 32-column row segments at 16-byte alignment.
template <typename T, typename M>
static bool bulk_ok(const VisitArgs<T, M>& a) {
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  return a.B % 32 == 0 && (a.ld * sizeof(M)) % 16 == 0 && al(a.f) &&
         (!a.u_src || al(a.u_src)) && (!a.uH || al(a.uH)) && (!a.uc || al(a.uc)) &&
         visit_bulk_enabled();
}

template <typename T, typename M, int SHAPE, int SRC, bool CR, bool EPI>
static void launch_visit_t(const VisitArgs<T, M>& a, cudaStream_t s) {
  const bool om1 = a.gc.omega == T(1);
  // bulk (TMA) staging pays off where per-lane LDGSTS saturates the MIO
  // queue: sources with >= 5 staged rows per pair (the FAS-correction visits);
  // measured slower than cp.async for 3-4 rows (profiles/r01 notes), and for
  // short chains (owned width < 64: levels 10-11 of config 2, where the lane-0
  // issue of five bulk copies per pair sits on the critical path)
  // Bulk copies only for scalar fp64 lanes: with two columns per lane (the
  // default for B % 64 == 0) per-lane 16-byte cp.async measured faster on
  // every config (config 2 / 4 / 5: +0.3 / +1.5 / +1.6 % per cycle), and fp32
  // lanes likewise (config 5 fp32: level-19 up 452 -> 379 us)
  constexpr bool bulk_lanes = std::is_same<T, double>::value && std::is_same<M, double>::value;
  // and only with more warps than SM sub-partitions: a warp issuing alone
  // waits on lane 0's serial bulk issue every pair (an 8-way shard of config 4,
  // U_23 with scalar lanes: 19 % of the stall samples on the mbarrier wait)
  const bool many = a.P * a.nrg > visit_smsps();
  const bool bulk = bulk_lanes && SrcRows<SRC, CR>::R >= 5 && a.W >= 64 && many && bulk_ok(a);
  // functional output of the final up visit (non-SR: FAS correction; SR: Pi + CR)
  if constexpr (!EPI && ((SRC == SRC_FMG && CR) || (SRC == SRC_CORR && !CR))) {
    if (a.fun_part) {
      if (om1) {
        if (bulk) launch_visit_k<T, M, SHAPE, SRC, CR, EPI, true, true, true>(a, s);
        else launch_visit_k<T, M, SHAPE, SRC, CR, EPI, true, false, true>(a, s);
      } else {
        if (bulk) launch_visit_k<T, M, SHAPE, SRC, CR, EPI, false, true, true>(a, s);
        else launch_visit_k<T, M, SHAPE, SRC, CR, EPI, false, false, true>(a, s);
      }
      return;
    }
  }
  if (om1) {
    if (bulk) launch_visit_k<T, M, SHAPE, SRC, CR, EPI, true, true>(a, s);
    else launch_visit_k<T, M, SHAPE, SRC, CR, EPI, true, false>(a, s);
  } else {
    if (bulk) launch_visit_k<T, M, SHAPE, SRC, CR, EPI, false, true>(a, s);
    else launch_visit_k<T, M, SHAPE, SRC, CR, EPI, false, false>(a, s);
  }
}


// Fill the kernel arguments for lane type TV (T, or V2<T>: two columns per
// lane) from a validated descriptor and launch.
// TM: the lane's storage type (TV, or the fp32 twin of an fp64 lane type
// under fp64 arithmetic); edge records (d.E, d.E_out) then hold TV values.
template <typename TV, typename T, int SHAPE, typename TM = TV>
void visit_fill_launch(const VisitDesc<T>& d, cudaStream_t s) {
  constexpr int C = LaneCols<TV>::value;
  auto cv = [](const T* p) { return reinterpret_cast<const TM*>(p); };
  auto mv = [](T* p) { return reinterpret_cast<TM*>(p); };
  auto rv = [](T* p) { return reinterpret_cast<TV*>(p); };
  VisitArgs<TV, TM> a;
  a.n = d.n;
  a.ld = d.ld / C;
  a.B = d.B / C;
  a.nrg = (a.B + 31) / 32;
  a.nc = d.n / 2;
  a.gc = make_coef<TV>(d.n, d.omega);
  a.inv_H2 = (TV)pow4(level_of(d.n) - 1);
  a.kz = make_kz<TV>(d.proj_diag);
  a.write_u = d.write_u;
  a.u_src = cv(d.u_src);
  a.uH = cv(d.uH);
  a.uc = cv(d.uc);
  a.f = cv(d.f);
  a.u_out = mv(d.u_out);
  a.uH_out = mv(d.uH_out);
  a.fH_out = mv(d.fH_out);
  a.E = rv(d.E);
  a.cnt = d.cnt;
  a.olo = d.olo;
  a.ohi = d.ohi;
  a.elo = d.elo;
  a.ehi = d.ehi;
  a.p_begin = 0;
  a.qlo = d.qlo >= 0 ? d.qlo : 0;
  a.qhi = d.qhi >= 0 ? d.qhi : a.nc - 1;
  a.E_out = rv(d.E_out);
  a.left_remote = d.left_remote;
  a.right_remote = d.right_remote;
  a.fun_w = cv(d.fun_w);
  a.fun_part = rv(d.fun_part);
  if (d.olo) {
    a.P = d.P;
    a.W = 0;
    a.b = 0;
  } else {
    a.W = d.W;
    a.b = d.b;
    a.P = d.n / d.W;
    if (d.p_count >= 0) {
      a.p_begin = d.p_begin;
      a.P = d.p_count;
    }
  }
  if (a.P == 0) return;
#define FMGSR_DISPATCH(SRCV)                                                    \
  if (d.cr) {                                                                  \
    if (d.epi) launch_visit_t<TV, TM, SHAPE, SRCV, true, true>(a, s);                     \
    else launch_visit_t<TV, TM, SHAPE, SRCV, true, false>(a, s);                          \
  } else {                                                                     \
    if (d.epi) launch_visit_t<TV, TM, SHAPE, SRCV, false, true>(a, s);                    \
    else launch_visit_t<TV, TM, SHAPE, SRCV, false, false>(a, s);                         \
  }
  if (d.src == SRC_LOAD) {
    FMGSR_DISPATCH(SRC_LOAD)
  } else if (d.src == SRC_CORR) {
    FMGSR_DISPATCH(SRC_CORR)
  } else {
    FMGSR_DISPATCH(SRC_FMG)
  }
#undef FMGSR_DISPATCH
}

}  // namespace fmgsr
