// kernels_group.cu -- level visits of SHORT patches (owned width W <= 8).
//
// On the mid levels of a deep hierarchy (config 4: levels 13-15, 4096 patches
// of 2-8 cells with an 8-cell buffer) a patch chain is 10-16 cells long, so
// the streaming visit_kernel is all head and tail: its ring staging, the
// general boundary step and one fence + counter round per patch cost ~2000
// instructions and ~18 k cycles per warp for ~1800 cycles of Gauss-Seidel
// (ncu, profiles/r02/mid_levels_config4.txt).  Here one CTA of four warps owns
// a GROUP of G consecutive patches x 32 RHS columns (one lane per column):
//   * the group's window (G W + b + 2 rows of u, f; the FAS-correction source
//     rows on an up visit) is fetched once, every row in flight at the same
//     time (cp.async into per-lane columns of shared memory, one wait), the
//     rows dealt round-robin to the warps;
//   * on an up visit the smoother input u + P(uH - R u) (cycles.py:120-121,
//     stencils.py:39-64) is built for the whole window in a data-parallel
//     pass -- the expressions of PairSource<SRC_CORR>::make;
//   * the G patch chains (additive smoother, _kernels_numba.py:60-92: every
//     patch starts from the same input) are independent, so they are dealt to
//     the warps and a lane runs IL of them interleaved -- the per-cell
//     arithmetic and order of each chain are the reference's, only the
//     schedule differs;
//   * restriction + tau (stencils.py:108-125) run over the group's smoothed
//     cells, a contiguous run of coarse cells per warp with the expressions of
//     Epilogue::push / finish, and only the GROUP boundaries go through the
//     edge-record protocol: one fence and counter round per G patches, and
//     any owned width >= 2 fuses (G W >= 4).
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

constexpr int GROUP_NT = 128;  // threads per group CTA (4 warps)

template <typename T, bool OMEGA1>
__device__ __forceinline__ T gs_interior(const GsCoef<T>& gc, T l, T u, T r, T f) {
  T s = xsub(xsub(xmul(T(2), u), l), r);
  T resid = xsub(f, xmul(gc.inv_h2, s));
  if (!OMEGA1) resid = xmul(gc.omega, resid);  // omega == 1: the product is exact
  return xadd(u, xmul(resid, gc.rdiag));
}

// One CTA of NW warps per (group, 32 RHS columns); one lane per column, the
// group's rows, chains and coarse cells dealt round-robin to the warps.
template <typename T, int SRC, bool EPI, bool OMEGA1, int IL>
__global__ void __launch_bounds__(GROUP_NT) group_visit_kernel(const GroupArgs<T> a) {
  extern __shared__ __align__(16) unsigned char group_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = GROUP_NT / 32;
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

  T* Us = reinterpret_cast<T*>(group_smem) + lane;  // row k of this column: Us[k * 32]
  T* Fs = Us + a.rows_u * 32;
  T* Hs = Fs + a.rows_f * 32;
  T* Ns = Hs + a.rows_h * 32;  // smoothed owned cells (EPI)
  i64 ubase;  // the cell held by row 0 of Us

  {
    const int nf = (int)(oe - wlo);
    const T* src = a.f + rr + (wlo + w) * ld;
    T* dst = Fs + w * 32;
    for (int k = w; k < nf; k += NW, src += NW * ld, dst += NW * 32) cp_async(dst, src);
  }
  if (SRC == SRC_LOAD) {
    ubase = ulo;
    const int nu = (int)(uhi - ulo);
    const T* src = a.u_src + rr + (ulo + w) * ld;
    T* dst = Us + w * 32;
    for (int k = w; k < nu; k += NW, src += NW * ld, dst += NW * 32) cp_async(dst, src);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  } else if (SRC == SRC_FMG) {
    // Pi(uH) on the pairs [q0, q1] (stencils.py:67-105): coarse cells q-2 .. q+2,
    // and the four cells next to a domain end for its special rows
    const i64 nc = a.nc;
    const i64 q0 = ulo >> 1, q1 = (uhi - 1) >> 1;
    i64 h0 = q0 - 2 > 0 ? q0 - 2 : 0, h1 = q1 + 2 < nc - 1 ? q1 + 2 : nc - 1;
    if (q0 <= 1 && h1 < 3) h1 = 3;            // rows 0-3 read c[0..3]
    if (q1 >= nc - 2 && h0 > nc - 4) h0 = nc - 4;  // rows nf-4..nf-1 read c[nc-4..nc-1]
    ubase = 2 * q0;
    const int nh = (int)(h1 - h0 + 1);
    {
      const T* sh = a.uH + rr + (h0 + w) * ld;
      for (int k = w; k < nh; k += NW, sh += NW * ld) cp_async(Hs + k * 32, sh);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    auto C = [&](i64 j) { return Hs[(int)(j - h0) * 32]; };
    for (i64 q = q0 + w; q <= q1; q += NW) {  // PairSource<SRC_FMG>::make, pair q
      T e, o;
      if (q >= 2 && q <= nc - 3) {
        const T c0 = C(q - 2), c1 = C(q - 1), c2 = C(q), c3 = C(q + 1), c4 = C(q + 2);
        e = xsub(xadd(xadd(xmul(T(-5), c0), xmul(T(35), c1)), xmul(T(105), c2)), xmul(T(7), c3));
        o = xsub(xadd(xadd(xmul(T(-7), c1), xmul(T(105), c2)), xmul(T(35), c3)), xmul(T(5), c4));
      } else if (q == 0) {  // rows 0, 1 over c[0..2]
        const T c2 = C(0), c3 = C(1), c4 = C(2);
        e = xsub(xmul(T(70), c2), xmul(T(2), c3));
        o = xsub(xadd(xmul(T(112), c2), xmul(T(35), c3)), xmul(T(5), c4));
      } else if (q == 1) {  // rows 2, 3 over c[0..3]
        const T c1 = C(0), c2 = C(1), c3 = C(2), c4 = C(3);
        e = xsub(xadd(xmul(T(40), c1), xmul(T(105), c2)), xmul(T(7), c3));
        o = xsub(xadd(xadd(xmul(T(-7), c1), xmul(T(105), c2)), xmul(T(35), c3)), xmul(T(5), c4));
      } else if (q == nc - 2) {  // rows nf-4, nf-3
        const T c0 = C(nc - 4), c1 = C(nc - 3), c2 = C(nc - 2), c3 = C(nc - 1);
        e = xsub(xadd(xadd(xmul(T(-7), c3), xmul(T(105), c2)), xmul(T(35), c1)), xmul(T(5), c0));
        o = xsub(xadd(xmul(T(40), c3), xmul(T(105), c2)), xmul(T(7), c1));
      } else {  // q == nc - 1: rows nf-2, nf-1
        const T c0 = C(nc - 3), c1 = C(nc - 2), c2 = C(nc - 1);
        e = xsub(xadd(xmul(T(112), c2), xmul(T(35), c1)), xmul(T(5), c0));
        o = xsub(xmul(T(70), c2), xmul(T(2), c1));
      }
      const int k = (int)(q - q0);
      Us[(2 * k) * 32] = xmul(e, T(0.0078125));  // x / 128 == x * 2^-7 exactly
      Us[(2 * k + 1) * 32] = xmul(o, T(0.0078125));
    }
    __syncthreads();
  } else {
    // u + P(uH - R u) on the pairs [q0, q1] needs c = uH - R u one pair further out
    const i64 nc = a.nc;
    const i64 q0 = ulo >> 1, q1 = (uhi - 1) >> 1;
    const i64 rq0 = q0 > 0 ? q0 - 1 : 0, rq1 = q1 < nc - 1 ? q1 + 1 : nc - 1;
    ubase = 2 * rq0;
    const int np = (int)(rq1 - rq0 + 1);
    {
      const T* su = a.u_src + rr + (2 * (rq0 + w)) * ld;
      const T* sh = a.uH + rr + (rq0 + w) * ld;
      for (int k = w; k < np; k += NW, su += 2 * NW * ld, sh += NW * ld) {
        cp_async(Us + (2 * k) * 32, su);
        cp_async(Us + (2 * k + 1) * 32, su + ld);
        cp_async(Hs + k * 32, sh);
      }
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    for (int k = w; k < np; k += NW)  // c_j = uH[j] - 0.5 (u[2j] + u[2j+1])
      Hs[k * 32] = xsub(Hs[k * 32], xmul(T(0.5), xadd(Us[(2 * k) * 32], Us[(2 * k + 1) * 32])));
    __syncthreads();
    const int k0 = (int)(q0 - rq0), k1 = (int)(q1 - rq0);
    for (int k = k0 + w; k <= k1; k += NW) {  // PairSource<SRC_CORR>::make, pair rq0 + k
      const i64 q = rq0 + k;
      const T s1 = Hs[k * 32], s2 = Us[(2 * k) * 32], s3 = Us[(2 * k + 1) * 32];
      const T p0v = (q == 0) ? xmul(T(0.5), s1)
                             : xmul(T(0.25), xadd(Hs[(k - 1) * 32], xmul(T(3), s1)));
      const T p1v = (q == nc - 1) ? xmul(T(0.5), s1)
                                  : xmul(T(0.25), xadd(xmul(T(3), s1), Hs[(k + 1) * 32]));
      Us[(2 * k) * 32] = xadd(s2, p0v);
      Us[(2 * k + 1) * 32] = xadd(s3, p1v);
    }
    __syncthreads();
  }

  // ---- the group's patch chains: IL per warp at a time ---------------------------
  const GsCoef<T> gc = a.gc;
  T* out = ((!EPI || a.write_u) && a.u_out) ? a.u_out + rr : nullptr;
  const int uo = (int)(os - ubase), fo = (int)(os - wlo);  // row of cell `os` in Us / Fs
  // interior groups: every smoothed cell has both neighbours and all IL-blocks are full
  const bool bnd = (os - b - 1 < 0) || (oe >= n) || (Gp % IL != 0);
  if (!bnd) {
    for (int k0 = w * IL; k0 < Gp; k0 += NW * IL) {
      T uL[IL];
      const T* up = Us + (uo + k0 * W - b) * 32;  // chain c: cell os + (k0 + c) W - b + t
      const T* fp = Fs + (fo + k0 * W - b) * 32;
      T cu[IL];  // the current cell's input: the right neighbour read one step earlier
#pragma unroll
      for (int c = 0; c < IL; c++) {
        uL[c] = up[(c * W - 1) * 32];
        cu[c] = up[(c * W) * 32];
      }
      for (int t = 0; t < b; t++) {  // buffer cells left of each patch
#pragma unroll
        for (int c = 0; c < IL; c++) {
          const int x = (c * W + t) * 32;
          const T nx = up[x + 32];
          uL[c] = gs_interior<T, OMEGA1>(gc, uL[c], cu[c], nx, fp[x]);
          cu[c] = nx;
        }
      }
      T* po = out ? out + (os + (i64)k0 * W) * ld : nullptr;
      T* pn = Ns + (k0 * W) * 32;
      for (int t = 0; t < W; t++) {  // owned cells
#pragma unroll
        for (int c = 0; c < IL; c++) {
          const int x = (c * W + b + t) * 32;
          const T nx = up[x + 32];
          const T v = gs_interior<T, OMEGA1>(gc, uL[c], cu[c], nx, fp[x]);
          uL[c] = v;
          cu[c] = nx;
          if (EPI) pn[(c * W + t) * 32] = v;
          if (po) po[(i64)(c * W + t) * ld] = v;
        }
      }
    }
  } else {
    // groups at a domain end or partly filled: the same chains, every cell
    // through the general gs_cell (domain rows first, as the reference)
    for (int k = w; k < Gp; k += NW) {
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
  __syncthreads();

  // ---- restriction + tau over the group's owned cells (stencils.py:108-125) ------
  // One coarse cell per (warp, step), each from the smoothed cells in Ns with
  // the expressions of Epilogue::push / finish; the first and last coarse cell
  // of the group need the neighbour group's cells: edge records, as visit_kernel.
  const T ih = gc.inv_h2, iH = a.inv_H2;
  const bool left_dom = (os == 0), right_dom = (oe == n);
  const i64 j0 = os >> 1;
  const int ncg = (int)((oe - os) >> 1);  // coarse cells of the group, >= 2
  const T* Fo = Fs + fo * 32;
  T* fH = a.fH_out + rr;
  T* uHo = a.uH_out ? a.uH_out + rr : nullptr;
  auto N = [&](int i) { return Ns[i * 32]; };                 // smoothed owned cell os + i
  auto Ru = [&](int c) { return xmul(T(0.5), xadd(N(2 * c), N(2 * c + 1))); };
  auto Lu = [&](int i) { return xmul(xsub(xsub(xmul(T(2), N(i)), N(i - 1)), N(i + 1)), ih); };
  if (w == 0) {
    // slab edges of a shard go to the outbox (the neighbour shard finishes them)
    EdgeRec<T> left, right;
    if (!left_dom) {
      left.v[0] = N(0);
      left.v[1] = N(1);
      left.v[2] = Lu(1);
      left.v[3] = Ru(1);
      left.v[4] = xmul(T(0.5), xadd(Fo[0], Fo[32]));
    }
    if (!right_dom) {
      const int s = 2 * ncg;
      right.v[0] = N(s - 2);
      right.v[1] = N(s - 1);
      right.v[2] = Lu(s - 2);
      right.v[3] = Ru(ncg - 2);
      right.v[4] = xmul(T(0.5), xadd(Fo[(s - 2) * 32], Fo[(s - 1) * 32]));
    }
    const i64 ldE = (i64)a.nrg * 32;
    const bool remL = !left_dom && g == 0 && a.left_remote;
    const bool remR = !right_dom && (i64)g == a.ngroups - 1 && a.right_remote;
    if (remL) {
#pragma unroll
      for (int k = 0; k < 5; k++) a.E_out[(0 * 5 + k) * ldE + r] = left.v[k];
    }
    if (remR) {
#pragma unroll
      for (int k = 0; k < 5; k++) a.E_out[(1 * 5 + k) * ldE + r] = right.v[k];
    }
    edge_arrive2<T, false, T>(a.E, a.cnt, ldE, a.nrg, lane, rg, r, true, fH, ld, ih, iH,
                              !left_dom && !remL, p0, left, os, !right_dom && !remR, p0 + Gp,
                              right, oe);
  }
  // a contiguous run of coarse cells per warp, sliding over the smoothed cells
  // (each read once); warp 0 (busy with the edge protocol) takes the last,
  // possibly short, run
  const int per = (ncg + NW - 1) / NW;
  const int cb = (NW - 1 - w) * per, ce = cb + per < ncg ? cb + per : ncg;
  if (cb >= ce) return;
  T nm1 = cb > 0 ? N(2 * cb - 1) : T(0), Rm = cb > 0 ? Ru(cb - 1) : T(0);
  T n0 = N(2 * cb), n1 = N(2 * cb + 1);
  T Rc = xmul(T(0.5), xadd(n0, n1));
  for (int c = cb; c < ce; c++) {
    T n2 = T(0), n3 = T(0), Rn = T(0);
    if (c + 1 < ncg) {
      n2 = N(2 * c + 2);
      n3 = N(2 * c + 3);
      Rn = xmul(T(0.5), xadd(n2, n3));
    }
    if (uHo) uHo[(j0 + c) * ld] = Rc;
    const T Le = xmul(xsub(xsub(xmul(T(2), n0), nm1), n1), ih);  // Lu at the pair's even cell
    const T Lo = xmul(xsub(xsub(xmul(T(2), n1), n0), n2), ih);   // ... and its odd cell
    T LH, RL;
    bool emit = true;
    if (c == 0) {
      emit = left_dom;  // otherwise completed through the edge records
      LH = xmul(xsub(xmul(T(3), Rc), Rn), iH);
      RL = xmul(T(0.5), xadd(xmul(xsub(xmul(T(3), n0), n1), ih), Lo));
    } else if (c == ncg - 1) {
      emit = right_dom;
      LH = xmul(xsub(xmul(T(3), Rc), Rm), iH);
      RL = xmul(T(0.5), xadd(Le, xmul(xsub(xmul(T(3), n1), n0), ih)));
    } else {
      LH = xmul(xsub(xsub(xmul(T(2), Rc), Rm), Rn), iH);
      RL = xmul(T(0.5), xadd(Le, Lo));
    }
    if (emit) {
      const T Rf = xmul(T(0.5), xadd(Fo[(2 * c) * 32], Fo[(2 * c + 1) * 32]));
      fH[(j0 + c) * ld] = xadd(Rf, xsub(LH, RL));
    }
    nm1 = n1;
    Rm = Rc;
    n0 = n2;
    n1 = n3;
    Rc = Rn;
  }
}

template <typename T, int SRC, bool EPI, bool OMEGA1, int IL>
void launch_group_k(const GroupArgs<T>& a, size_t smem, cudaStream_t s) {
  auto k = group_visit_kernel<T, SRC, EPI, OMEGA1, IL>;
  if (smem > 48 * 1024)
    require(smem <= (size_t)smem_optin((const void*)k), "group visit: shared memory budget exceeded");
  k<<<(unsigned)(a.ngroups * a.nrg), GROUP_NT, smem, s>>>(a);
}

template <typename T, int SRC, bool EPI>
void launch_group_il(const GroupArgs<T>& a, size_t smem, cudaStream_t s) {
  const bool om1 = a.gc.omega == T(1);
  const int per_warp = a.G / (GROUP_NT / 32);  // chains per warp (G is a power of two)
  const int il = per_warp >= 4 ? 4 : per_warp >= 2 ? 2 : 1;
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

// widest owned width served here (FMGSR_GROUP_MAXW overrides, for A/B runs)
int group_max_w() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_GROUP_MAXW");
    v = e ? atoi(e) : 8;
    if (v > 16) v = 16;
  }
  return v;
}

}  // namespace

// FMGSR_VISIT_GROUP=0 keeps every visit on the streaming kernel (A/B runs)
bool group_visit_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_VISIT_GROUP");
    v = (e && std::string(e) == "0") ? 0 : 1;
  }
  return v == 1;
}

// Short-patch visits (FMG-prolongation top visits and plain-load down visits,
// each with or without the fused restriction, FAS-correction up visits; no
// Kaczmarz pass, uniform geometry).
// Returns false when the visit is not of that kind: the caller then uses the
// streaming kernel.
template <typename T>
bool try_group_visit(const VisitDesc<T>& d, cudaStream_t s) {
  if (!group_visit_enabled() || d.olo || d.cr || d.fun_part || d.f64_arith) return false;
  if (!(d.src == SRC_LOAD || d.src == SRC_FMG || (d.src == SRC_CORR && !d.epi))) return false;
  // W = 16 measured slower than the streaming kernel (config 4 level 16: 49 / 42 us
  // against 40 / 33 us per down / up visit): two chains per group leave two of
  // the four warps without chain work
  if (d.W < 2 || d.W > group_max_w() || (d.W & (d.W - 1)) != 0 || d.b < 0 || d.b > 32 || d.n < 8) return false;
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
  a.rows_h = d.src == SRC_LOAD ? 0 : a.rows_u / 2 + (d.src == SRC_FMG ? 8 : 0);
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
  } else if (d.src == SRC_FMG) {
    if (d.epi) launch_group_il<T, SRC_FMG, true>(a, smem, s);
    else launch_group_il<T, SRC_FMG, false>(a, smem, s);
  } else {
    launch_group_il<T, SRC_CORR, false>(a, smem, s);
  }
  check_launch("group_visit_kernel");
  return true;
}

template bool try_group_visit<double>(const VisitDesc<double>&, cudaStream_t);
template bool try_group_visit<float>(const VisitDesc<float>&, cudaStream_t);

}  // namespace fmgsr
