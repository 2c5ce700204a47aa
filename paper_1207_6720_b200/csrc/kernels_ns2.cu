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
#include <cstdlib>
#include <string>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

// the fills live in kernels_ns2_{d,f,v2d,v2f}.cu (one lane type each)
template <typename TV, typename T>
void ns2_fill_launch(const Ns2Desc<T>& d, cudaStream_t s);

// FMGSR_NS2_CPL=1 forces one RHS column per lane (A/B tests)
static bool ns2_cpl2_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FMGSR_NS2_CPL");
    v = (e && std::string(e) == "1") ? 0 : 1;
  }
  return v == 1;
}

// Two RHS columns per lane (V2 lanes, as in the visit kernel): whole
// 64-column groups, 2-element-aligned rows, pointers and scratch stride.
// Only for the FAS-correction (U) visits of long chains: measured on config 3
// (tools/visit_breakdown.py, FMGSR_NS2_CPL=1 vs default) those gain 4-6 % at
// W >= 256 (levels 16-19), while the Pi-sourced T / SR-up visits lose 4-9 %
// and every visit with W < 256 loses up to 35 % -- the Newton-GS chain wants
// more resident warps (16 per SM with scalar lanes, 8 with V2 lanes at
// ~215 registers) rather than two interleaved chains per lane.
template <typename T>
static bool ns2_cpl2_ok(const Ns2Desc<T>& d) {
  constexpr uintptr_t A = 2 * sizeof(T);
  auto al = [](const void* p) { return ((uintptr_t)p & (A - 1)) == 0; };
  if (d.src != SRC_CORR || d.W < 256) return false;
  return ns2_cpl2_enabled() && d.B % 64 == 0 && d.ld % 2 == 0 && d.sld % 2 == 0 &&
         al(d.u_src) && al(d.uH) && al(d.uc) && al(d.f) && al(d.u_out) && al(d.scratch) &&
         al(d.uH_out) && al(d.fH_out) && al(d.E);
}

template <typename T>
void launch_smooth_ns2(const Ns2Desc<T>& d, cudaStream_t s) {
  require(d.n >= 8 && is_pow2(d.n), "ns2: level size must be a power of two >= 8");
  require(d.W >= 2 && d.W % 2 == 0 && d.n % d.W == 0, "ns2: owned width must be even and divide n");
  require((d.u_out || (d.epi && !d.write_u)) && d.f && d.scratch, "ns2: null pointer");
  require(d.sld >= (i64)((d.B + 31) / 32) * 32, "ns2: scratch stride too small");
  if (d.src == SRC_LOAD) require(d.u_src != nullptr, "ns2: LOAD needs u_src");
  if (d.src == SRC_CORR) require(d.u_src && d.uH, "ns2: CORR needs u_src and uH");
  if (d.src == SRC_FMG) require(d.uH != nullptr, "ns2: FMG needs uH");
  if (d.cr && d.src != SRC_FMG) require(d.uc != nullptr, "ns2: CR needs uc");
  if (d.epi) {
    require(!d.cr && (d.src == SRC_FMG || d.src == SRC_LOAD), "ns2: fused restriction only on T / D visits");
    require(d.W >= 4 && d.fH_out && d.E && d.cnt, "ns2: epilogue needs W >= 4 and its buffers");
  }
  if (ns2_cpl2_ok(d)) ns2_fill_launch<V2<T>>(d, s);
  else ns2_fill_launch<T>(d, s);
  check_launch("ns2_kernel");
}

template void launch_smooth_ns2<double>(const Ns2Desc<double>&, cudaStream_t);
template void launch_smooth_ns2<float>(const Ns2Desc<float>&, cudaStream_t);

}  // namespace fmgsr
