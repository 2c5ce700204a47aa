// kernels_visit_mp.cu -- FAS-correction up visits with several patches per warp.
//
// On the large levels of a many-patch hierarchy (config 4: 4096 two-column
// warps per visit over 2368 resident warp slots) a warp of the streaming
// visit_kernel lives for one patch: every patch pays the chain head (the
// first loads' latency) and the launch fills 1.7 waves.  An up visit has no
// epilogue and no cross-warp protocol, so a warp can simply run PPW
// consecutive patches one after the other with the same Chain -- the
// arithmetic of every chain is untouched, there are PPW times fewer, longer
// lived warps (one wave), and the next patch's head loads hit rows the warp
// has just streamed.  Measured on config 4 (profiles/r02/ab_up_ppw): level-17..20
// up visits 1.5-6 % faster with 4 patches per warp, levels 22-23 2 % slower
// (so only patches of 32-256 cells run this way).  Down visits lose with the
// same change (half the warps leave the 4-pair ring too little in flight, and
// the edge records a warp must park spill its 128 registers), so they keep
// one patch per warp; this kernel is the up visit only, in its own
// translation unit so visit_kernel's code is unchanged.
#include <cstdlib>
#include <string>

#include "visit_impl.cuh"

namespace fmgsr {

namespace {

template <typename T, bool OMEGA1, int NT, int D, int PPW>
__global__ void __launch_bounds__(NT, (D <= 4 ? 512 : 256) / NT)
    visit_up_mp_kernel(const VisitArgs<T, T> a) {
  extern __shared__ __align__(128) unsigned char visit_mp_smem[];
  const int lane = threadIdx.x & 31;
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nrg = (unsigned)a.nrg;
  const unsigned pg32 = nrg == 1 ? gw : gw / nrg;  // run of PPW patches
  const int rg = (int)(gw - pg32 * nrg);
  const i64 pl_first = (i64)pg32 * PPW;
  if (pl_first >= a.P) return;  // warp-uniform
  const int npw = (int)(a.P - pl_first < (i64)PPW ? a.P - pl_first : (i64)PPW);
  const int r = rg * 32 + lane;
  const int rr = r < a.B ? r : a.B - 1;  // as visit_kernel: every store unconditional

  Chain<T, SRC_CORR, false, false, OMEGA1, NT, D, false, false, T> ch;
  ch.lane = lane;
  ch.bars = nullptr;
  ch.src.u = a.u_src + rr;
  ch.src.uH = a.uH + rr;
  ch.src.uc = nullptr;
  ch.src.f = a.f + rr;
  ch.src.ld = a.ld;
  ch.src.nc = a.nc;
  ch.src.kz = a.kz;
  ch.src.qlo = a.qlo;
  ch.src.qhi = a.qhi;
  ch.gc = a.gc;
  ch.n = a.n;
  ch.nc = a.nc;
  ch.ld = a.ld;
  ch.store = true;
  ch.ring = reinterpret_cast<T*>(visit_mp_smem) + threadIdx.x;
  ch.out = a.u_out + rr;
  ch.fw = nullptr;
  ch.facc = T(0);
  ch.epi = nullptr;
  for (int g = 0; g < npw; g++) {
    const i64 p = a.p_begin + pl_first + g;
    const i64 os = p * a.W, oe = os + a.W;
    const i64 ws = os - a.b > 0 ? os - a.b : 0;
    const i64 we = oe + a.b < a.n ? oe + a.b : a.n;
    ch.src.wlo = ws >> 1;
    ch.src.whi = we >> 1;
    ch.ws = ws;
    ch.os = os;
    ch.oe = oe;
    ch.run(we);  // ends with cp.async.wait_group 0: the ring is free for the next patch
  }
}

template <int SHAPE, int PPW>
void launch_mp(const VisitArgs<V2<double>, V2<double>>& a, cudaStream_t s) {
  using T = V2<double>;
  constexpr int NT = VisitShape<SHAPE>::NT, D = VisitShape<SHAPE>::D;
  constexpr size_t smem = visit_smem_bytes<T, SRC_CORR, false, NT, D>();
  const bool om1 = a.gc.omega == T(1);
  const i64 warps = ((a.P + PPW - 1) / PPW) * a.nrg;
  const i64 blocks = (warps + NT / 32 - 1) / (NT / 32);
  if (om1) {
    auto k = visit_up_mp_kernel<T, true, NT, D, PPW>;
    if (smem > 48 * 1024)
      require(smem <= (size_t)smem_optin((const void*)k), "visit: shared memory budget exceeded");
    k<<<(unsigned)blocks, NT, smem, s>>>(a);
  } else {
    auto k = visit_up_mp_kernel<T, false, NT, D, PPW>;
    if (smem > 48 * 1024)
      require(smem <= (size_t)smem_optin((const void*)k), "visit: shared memory budget exceeded");
    k<<<(unsigned)blocks, NT, smem, s>>>(a);
  }
}

// patches per warp: FMGSR_VISIT_UP_PPW = 1 (off), 2, 4; default automatic
int up_ppw_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("FMGSR_VISIT_UP_PPW");
    v = e ? atoi(e) : -1;
  }
  return v;
}

}  // namespace

// FAS-correction up visit (SRC_CORR, no Kaczmarz pass, no epilogue, field
// output) with two-column fp64 lanes and uniform geometry -- the caller has
// checked visit_cpl2_ok(d).  Returns false when one patch per warp is the
// better shape: the caller then launches visit_kernel.
bool visit_up_mp(const VisitDesc<double>& d, bool r4, cudaStream_t s) {
  if (d.src != SRC_CORR || d.cr || d.epi || d.fun_part || d.olo || d.f64_arith || !d.u_out)
    return false;
  const i64 P = d.p_count >= 0 ? d.p_count : d.n / d.W;
  const i64 nrg = (d.B / 2 + 31) / 32;
  int ppw = up_ppw_env();
  if (ppw < 0) {
    // only where one patch per warp overfills the GPU's warp slots (16 per SM at
    // the R4 shape): then PPW-times fewer warps still give every SM sub-partition
    // its share.  Short patches go to the group kernel before this is reached.
    // Patches of 32-256 cells: longer ones stream well as they are (config 4
    // level 23, 2048-cell patches: 2205 -> 2257 us with 4 per warp; level 19,
    // 128 cells: 165 -> 158 us).
    ppw = (P * nrg >= 4 * (i64)visit_smsps() && d.W >= 32 && d.W <= 256) ? 4 : 1;
  }
  if (ppw != 2 && ppw != 4) return false;
  using T = V2<double>;
  VisitArgs<T, T> a;
  a.n = d.n;
  a.ld = d.ld / 2;
  a.B = d.B / 2;
  a.nrg = (a.B + 31) / 32;
  a.nc = d.n / 2;
  a.gc = make_coef<T>(d.n, d.omega);
  a.inv_H2 = (T)pow4(level_of(d.n) - 1);
  a.kz = make_kz<T>(d.proj_diag);
  a.write_u = true;
  a.u_src = reinterpret_cast<const T*>(d.u_src);
  a.uH = reinterpret_cast<const T*>(d.uH);
  a.uc = nullptr;
  a.f = reinterpret_cast<const T*>(d.f);
  a.u_out = reinterpret_cast<T*>(d.u_out);
  a.uH_out = nullptr;
  a.fH_out = nullptr;
  a.E = nullptr;
  a.cnt = nullptr;
  a.olo = a.ohi = a.elo = a.ehi = nullptr;
  a.qlo = d.qlo >= 0 ? d.qlo : 0;
  a.qhi = d.qhi >= 0 ? d.qhi : a.nc - 1;
  a.E_out = nullptr;
  a.left_remote = a.right_remote = false;
  a.fun_w = nullptr;
  a.fun_part = nullptr;
  a.W = d.W;
  a.b = d.b;
  a.p_begin = d.p_count >= 0 ? d.p_begin : 0;
  a.P = P;
  if (a.P == 0) return true;
  if (r4) {
    if (ppw == 4) launch_mp<SHAPE_R4, 4>(a, s);
    else launch_mp<SHAPE_R4, 2>(a, s);
  } else {
    if (ppw == 4) launch_mp<SHAPE_WIDE, 4>(a, s);
    else launch_mp<SHAPE_WIDE, 2>(a, s);
  }
  return true;
}

}  // namespace fmgsr
