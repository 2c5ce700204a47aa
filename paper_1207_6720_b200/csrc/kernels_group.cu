// kernels_group.cu -- level visits of SHORT patches (owned width W <= 16).
//
// On the mid levels of a deep hierarchy (config 4: levels 13-16, 4096 patches
// of 2-16 cells with an 8-cell buffer) a patch chain is 10-24 cells long, so
// the streaming visit_kernel is all head and tail: its ring staging, the
// general boundary step and one fence + counter round per patch cost ~2000
// instructions and ~18 k cycles per warp for ~1800 cycles of Gauss-Seidel
// (ncu, profiles/r02/mid_levels_config4.txt).  Here one warp owns a GROUP of G
// consecutive patches x 32 RHS columns instead:
//   * the group's window (G W + b + 2 rows of u, f; the FAS-correction source
//     rows on an up visit) is fetched once, every row in flight at the same
//     time (cp.async into a per-lane column of shared memory, one wait);
//   * on an up visit the smoother input u + P(uH - R u) (cycles.py:120-121,
//     stencils.py:39-64) is built for the whole window in a data-parallel
//     pass -- the expressions of PairSource<SRC_CORR>::make;
//   * the G patch chains (additive smoother, _kernels_numba.py:60-92: every
//     patch starts from the same input) are independent, so a lane runs IL of
//     them interleaved -- the per-cell arithmetic and order of each chain are
//     the reference's, only the schedule differs;
//   * restriction + tau (stencils.py:108-125) run over the group's smoothed
//     cells with the Epilogue of the streaming kernel, and only the GROUP
//     boundaries go through the edge-record protocol: one fence and counter
//     round per G patches, and any owned width >= 2 fuses (G W >= 4).
// Edge records, counters and the shard outbox keep the streaming kernel's
// layout and indices (boundary = absolute patch index), so both kernels can
// serve different visits of one level.
#include <cstdlib>
#include <string>
#include <type_traits>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"
#include "visit_common.cuh"

namespace fmgsr {

namespace {

template <typename T>
struct GroupArgs {
  i64 n, ld, nc, p_begin, P, ngroups;
  int W, b, G, B, nrg;
  int rows_u, rows_f, rows_h;  // shared-memory rows per array (x 32 lanes)
  GsCoef<T> gc;
  T inv_H2;
  bool write_u, left_remote, right_remote;
  const T *u_src, *uH, *f;
  T *u_out, *uH_out, *fH_out, *E, *E_out;
  int* cnt;
};

template <typename T, bool OMEGA1>
__device__ __forceinline__ T gs_interior(const GsCoef<T>& gc, T l, T u, T r, T f) {
  T s = xsub(xsub(xmul(T(2), u), l), r);
  T resid = xsub(f, xmul(gc.inv_h2, s));
  if (!OMEGA1) resid = xmul(gc.omega, resid);  // omega == 1: the product is exact
  return xadd(u, xmul(resid, gc.rdiag));
}

// One warp per (group, 32 RHS columns); one lane per column.
template <typename T, int SRC, bool EPI, bool OMEGA1, int IL>
__global__ void __launch_bounds__(32) group_visit_kernel(const GroupArgs<T> a) {
  extern __shared__ __align__(16) unsigned char group_smem[];
  const int lane = threadIdx.x;
  const unsigned nrg = (unsigned)a.nrg;
  const unsigned g = nrg == 1 ? blockIdx.x : blockIdx.x / nrg;
  const int rg = (int)(blockIdx.x - g * nrg);
  const int r = rg * 32 + lane;
  // lanes past the last column run column B-1's chains and store its
  // bit-identical values (as visit_kernel): every store is unconditional
  const int rr = r < a.B ? r : a.B - 1;
  const i64 n = a.n, ld = a.ld;
  const int W = a.W, b = a.b;
  const i64 p0 = a.p_begin + (i64)g * a.G;
  const i64 pend = a.p_begin + a.P;
  const int Gp = (int)((pend - p0) < (i64)a.G ? (pend - p0) : (i64)a.G);
  const i64 os = p0 * W, oe = (p0 + Gp) * W;  // the group's owned cells
  const i64 wlo = os - b > 0 ? os - b : 0;    // first smoothed cell
  const i64 ulo = wlo > 0 ? wlo - 1 : 0;      // smoother input rows [ulo, uhi)
  const i64 uhi = oe < n ? oe + 1 : n;

  T* Us = reinterpret_cast<T*>(group_smem) + lane;  // row k of this lane: Us[k * 32]
  T* Fs = Us + a.rows_u * 32;
  T* Hs = Fs + a.rows_f * 32;
  T* Ns = Hs + a.rows_h * 32;  // smoothed owned cells (EPI)
  const T* f = a.f + rr;
  i64 ubase;  // the cell held by row 0 of Us

  for (i64 i = wlo; i < oe; i++) cp_async(Fs + (int)(i - wlo) * 32, f + i * ld);
  if (SRC == SRC_LOAD) {
    const T* u = a.u_src + rr;
    ubase = ulo;
    for (i64 i = ulo; i < uhi; i++) cp_async(Us + (int)(i - ulo) * 32, u + i * ld);
    cp_commit();
    cp_wait<0>();
  } else {
    // u + P(uH - R u) on the pairs [q0, q1] needs c = uH - R u one pair further out
    const T* u = a.u_src + rr;
    const T* uH = a.uH + rr;
    const i64 nc = a.nc;
    const i64 q0 = ulo >> 1, q1 = (uhi - 1) >> 1;
    const i64 rq0 = q0 > 0 ? q0 - 1 : 0, rq1 = q1 < nc - 1 ? q1 + 1 : nc - 1;
    ubase = 2 * rq0;
    for (i64 j = rq0; j <= rq1; j++) {
      const int k = (int)(j - rq0);
      cp_async(Us + (2 * k) * 32, u + (2 * j) * ld);
      cp_async(Us + (2 * k + 1) * 32, u + (2 * j + 1) * ld);
      cp_async(Hs + k * 32, uH + j * ld);
    }
    cp_commit();
    cp_wait<0>();
    const int np = (int)(rq1 - rq0 + 1);
    for (int k = 0; k < np; k++)  // c_j = uH[j] - 0.5 (u[2j] + u[2j+1])
      Hs[k * 32] = xsub(Hs[k * 32], xmul(T(0.5), xadd(Us[(2 * k) * 32], Us[(2 * k + 1) * 32])));
    for (i64 q = q0; q <= q1; q++) {  // PairSource<SRC_CORR>::make, pair q
      const int k = (int)(q - rq0);
      const T s1 = Hs[k * 32], s2 = Us[(2 * k) * 32], s3 = Us[(2 * k + 1) * 32];
      const T p0v = (q == 0) ? xmul(T(0.5), s1)
                             : xmul(T(0.25), xadd(Hs[(k - 1) * 32], xmul(T(3), s1)));
      const T p1v = (q == nc - 1) ? xmul(T(0.5), s1)
                                  : xmul(T(0.25), xadd(xmul(T(3), s1), Hs[(k + 1) * 32]));
      Us[(2 * k) * 32] = xadd(s2, p0v);
      Us[(2 * k + 1) * 32] = xadd(s3, p1v);
    }
  }

  // ---- the group's patch chains, IL at a time ------------------------------------
  const GsCoef<T> gc = a.gc;
  T* out = ((!EPI || a.write_u) && a.u_out) ? a.u_out + rr : nullptr;
  const int uo = (int)(os - ubase), fo = (int)(os - wlo);  // row of cell `os` in Us / Fs
  // interior groups: every smoothed cell has both neighbours and all IL-blocks are full
  const bool bnd = (os - b - 1 < 0) || (oe >= n) || (Gp % IL != 0);
  if (!bnd) {
    for (int k0 = 0; k0 < Gp; k0 += IL) {
      T uL[IL];
      const T* up = Us + (uo + k0 * W - b) * 32;  // chain c: cell os + (k0 + c) W - b + t
      const T* fp = Fs + (fo + k0 * W - b) * 32;
#pragma unroll
      for (int c = 0; c < IL; c++) uL[c] = up[(c * W - 1) * 32];
      for (int t = 0; t < b; t++) {  // buffer cells left of each patch
#pragma unroll
        for (int c = 0; c < IL; c++) {
          const int x = (c * W + t) * 32;
          uL[c] = gs_interior<T, OMEGA1>(gc, uL[c], up[x], up[x + 32], fp[x]);
        }
      }
      for (int t = b; t < b + W; t++) {  // owned cells
#pragma unroll
        for (int c = 0; c < IL; c++) {
          const int x = (c * W + t) * 32;
          const T v = gs_interior<T, OMEGA1>(gc, uL[c], up[x], up[x + 32], fp[x]);
          uL[c] = v;
          const int oc = (k0 + c) * W + t - b;  // owned cell index within the group
          if (EPI) Ns[oc * 32] = v;
          if (out) out[(os + oc) * ld] = v;
        }
      }
    }
  } else {
    // groups at a domain end or partly filled: the same chains, every cell
    // through the general gs_cell (domain rows first, as the reference)
    for (int k = 0; k < Gp; k++) {
      const i64 pos = os + (i64)k * W;
      const i64 ws = pos - b > 0 ? pos - b : 0;
      T uL = ws > 0 ? Us[(int)(ws - 1 - ubase) * 32] : T(0);
      for (i64 i = ws; i < pos + W; i++) {
        const T cur = Us[(int)(i - ubase) * 32];
        const T nxt = i + 1 < n ? Us[(int)(i + 1 - ubase) * 32] : T(0);
        const T v = gs_cell(gc, i, n, uL, cur, nxt, Fs[(int)(i - wlo) * 32]);
        uL = v;
        if (i >= pos) {
          if (EPI) Ns[(int)(i - os) * 32] = v;
          if (out) out[i * ld] = v;
        }
      }
    }
  }
  if (!EPI) return;

  // ---- restriction + tau over the group's owned pairs ----------------------------
  Epilogue<T, T> ep;
  ep.inv_h2 = gc.inv_h2;
  ep.inv_H2 = a.inv_H2;
  ep.left_dom = (os == 0);
  ep.right_dom = (oe == n);
  ep.write_uH = a.uH_out != nullptr;
  ep.uH_out = a.uH_out ? a.uH_out + rr : nullptr;
  ep.fH_out = a.fH_out + rr;
  ep.ld = ld;
  ep.nc = a.nc;
  ep.cnt = 0;
  ep.up2 = ep.up1 = ep.Lprev = ep.Rm2 = ep.Rm1 = ep.Rfm1 = T(0);
  const i64 j0 = os >> 1;
  const int npair = (int)((oe - os) >> 1);  // >= 2 (G W >= 4)
  const T* Fo = Fs + fo * 32;
  ep.push(j0, Ns[0], Ns[32], Fo[0], Fo[32], true);
  ep.push(j0 + 1, Ns[2 * 32], Ns[3 * 32], Fo[2 * 32], Fo[3 * 32], true);
  ep.fast_begin(j0 + 2);
  if (ep.write_uH) {
    for (int k = 2; k < npair; k++)
      ep.template push_fast<true>(Ns[(2 * k) * 32], Ns[(2 * k + 1) * 32], Fo[(2 * k) * 32],
                                  Fo[(2 * k + 1) * 32]);
  } else {
    for (int k = 2; k < npair; k++)
      ep.template push_fast<false>(Ns[(2 * k) * 32], Ns[(2 * k + 1) * 32], Fo[(2 * k) * 32],
                                   Fo[(2 * k + 1) * 32]);
  }
  EdgeRec<T> right;
  ep.finish(true, right);
  const i64 ldE = (i64)a.nrg * 32;
  // slab edges of a shard go to the outbox (the neighbour shard finishes them)
  const bool remL = !ep.left_dom && g == 0 && a.left_remote;
  const bool remR = !ep.right_dom && (i64)g == a.ngroups - 1 && a.right_remote;
  if (remL) {
#pragma unroll
    for (int k = 0; k < 5; k++) a.E_out[(0 * 5 + k) * ldE + r] = ep.left.v[k];
  }
  if (remR) {
#pragma unroll
    for (int k = 0; k < 5; k++) a.E_out[(1 * 5 + k) * ldE + r] = right.v[k];
  }
  edge_arrive2<T, false, T>(a.E, a.cnt, ldE, a.nrg, lane, rg, r, true, ep.fH_out, ld, ep.inv_h2,
                            ep.inv_H2, !ep.left_dom && !remL, p0, ep.left, os,
                            !ep.right_dom && !remR, p0 + Gp, right, oe);
}

template <typename T, int SRC, bool EPI, bool OMEGA1, int IL>
void launch_group_k(const GroupArgs<T>& a, size_t smem, cudaStream_t s) {
  auto k = group_visit_kernel<T, SRC, EPI, OMEGA1, IL>;
  if (smem > 48 * 1024)
    require(smem <= (size_t)smem_optin((const void*)k), "group visit: shared memory budget exceeded");
  k<<<(unsigned)(a.ngroups * a.nrg), 32, smem, s>>>(a);
}

template <typename T, int SRC, bool EPI>
void launch_group_il(const GroupArgs<T>& a, size_t smem, cudaStream_t s) {
  const bool om1 = a.gc.omega == T(1);
  const int il = a.G >= 4 ? 4 : a.G;
#define FMGSR_GROUP_IL(ILV)                                              \
  if (om1) launch_group_k<T, SRC, EPI, true, ILV>(a, smem, s);           \
  else launch_group_k<T, SRC, EPI, false, ILV>(a, smem, s);
  if (il == 4) {
    FMGSR_GROUP_IL(4)
  } else if (il == 2) {
    FMGSR_GROUP_IL(2)
  } else {
    FMGSR_GROUP_IL(1)
  }
#undef FMGSR_GROUP_IL
}

// FMGSR_VISIT_GROUP=0 keeps every visit on the streaming kernel (A/B runs)
bool group_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_VISIT_GROUP");
    v = (e && std::string(e) == "0") ? 0 : 1;
  }
  return v == 1;
}

}  // namespace

// Short-patch visits (plain-load down visits with or without the fused
// restriction, FAS-correction up visits; no Kaczmarz pass, uniform geometry).
// Returns false when the visit is not of that kind: the caller then uses the
// streaming kernel.
template <typename T>
bool try_group_visit(const VisitDesc<T>& d, cudaStream_t s) {
  if (!group_enabled() || d.olo || d.cr || d.fun_part || d.f64_arith) return false;
  if (!(d.src == SRC_LOAD || (d.src == SRC_CORR && !d.epi))) return false;
  if (d.W < 2 || d.W > 16 || (d.W & (d.W - 1)) != 0 || d.b < 0 || d.b > 32 || d.n < 8) return false;
  const i64 Plev = d.n / d.W;
  const i64 P = d.p_count >= 0 ? d.p_count : Plev;
  if (P == 0) return true;  // nothing to do
  const int nrg = (d.B + 31) / 32;
  // patches per group: up to 32 owned cells per group, fewer when that would
  // leave SM sub-partitions without a warp; the fused restriction needs >= 4 cells
  int G = (int)(32 / d.W);
  while (G > 1 && ((P + G - 1) / G) * nrg < (i64)visit_smsps() && (G / 2) * d.W >= 4) G /= 2;
  if (d.epi && (i64)G * d.W < 4) return false;
  if (d.epi && P * d.W < 4) return false;
  GroupArgs<T> a;
  a.n = d.n;
  a.ld = d.ld;
  a.nc = d.n / 2;
  a.p_begin = d.p_count >= 0 ? d.p_begin : 0;
  a.P = P;
  a.G = G;
  a.ngroups = (P + G - 1) / G;
  // the last group of an epilogue launch must own >= 4 cells too
  if (d.epi && (P - (a.ngroups - 1) * G) * d.W < 4) return false;
  a.W = (int)d.W;
  a.b = (int)d.b;
  a.B = d.B;
  a.nrg = nrg;
  const int gw = G * a.W;
  a.rows_f = gw + a.b;
  a.rows_u = d.src == SRC_LOAD ? gw + a.b + 2 : gw + a.b + 10;
  a.rows_h = d.src == SRC_LOAD ? 0 : a.rows_u / 2;
  a.gc = make_coef<T>(d.n, d.omega);
  a.inv_H2 = (T)pow4(level_of(d.n) - 1);
  a.write_u = d.write_u;
  a.left_remote = d.left_remote;
  a.right_remote = d.right_remote;
  a.u_src = d.u_src;
  a.uH = d.uH;
  a.f = d.f;
  a.u_out = d.u_out;
  a.uH_out = d.uH_out;
  a.fH_out = d.fH_out;
  a.E = d.E;
  a.E_out = d.E_out;
  a.cnt = d.cnt;
  const size_t smem =
      (size_t)(a.rows_u + a.rows_f + a.rows_h + (d.epi ? gw : 0)) * 32 * sizeof(T);
  if (smem > 100 * 1024) return false;
  if (d.src == SRC_LOAD) {
    if (d.epi) launch_group_il<T, SRC_LOAD, true>(a, smem, s);
    else launch_group_il<T, SRC_LOAD, false>(a, smem, s);
  } else {
    launch_group_il<T, SRC_CORR, false>(a, smem, s);
  }
  check_launch("group_visit_kernel");
  return true;
}

template bool try_group_visit<double>(const VisitDesc<double>&, cudaStream_t);
template bool try_group_visit<float>(const VisitDesc<float>&, cudaStream_t);

}  // namespace fmgsr
