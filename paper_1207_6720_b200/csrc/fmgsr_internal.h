// fmgsr_internal.h -- host-side internals shared by the translation units of
// libfmgsr_cuda.so: error reporting for the C ABI and the launcher templates.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace fmgsr {

typedef int64_t i64;

// Thrown by launchers and validators; turned into a negative return code and
// the text behind fmgsr_last_error() at the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum { ERR_ARG = -1, ERR_CUDA = -2, ERR_INTERNAL = -3 };

void set_last_error(const std::string& msg);
void clear_last_error();

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void check_launch(const char* what) { check_cuda(cudaGetLastError(), what); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(ERR_ARG, msg);
}

// Opt kernel `kf` into the device's full dynamic shared memory (the opt-in
// limit minus the kernel's static shared memory) on the CURRENT device --
// function attributes live per device context -- once per (device, kernel);
// returns the granted bytes (capi.cu).
int smem_optin(const void* kf);

__host__ __device__ inline double __longlong_as_double_hd(long long b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double d;
  __builtin_memcpy(&d, &b, sizeof d);
  return d;
#endif
}
__host__ __device__ inline int level_of(i64 n) {
  int k = 0;
  while (((i64)1 << (k + 1)) <= n) k++;
  return k;
}
// 4^k = h^-2 of level k as an exact double (2^(2k) built from its exponent
// bits; an integer shift would overflow for k >= 32)
__host__ __device__ inline double pow4(int k) {
  return __longlong_as_double_hd((long long)(1023 + 2 * k) << 52);
}
// launch shapes of the visit kernel (visit_impl.cuh VisitShape)
enum { SHAPE_WIDE = 0, SHAPE_DEEP = 1, SHAPE_R4 = 2 };
// SM sub-partitions (4 per SM) of the current device (kernels_visit.cu)
int visit_smsps();
// the short-patch group kernel (kernels_group.cu) is in use (FMGSR_VISIT_GROUP != 0)
bool group_visit_enabled();
inline bool is_pow2(i64 n) { return n >= 1 && (n & (n - 1)) == 0; }

// Run f(); map exceptions to C return codes.
template <typename F>
int guarded(F&& f) {
  try {
    clear_last_error();
    f();
    return 0;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ERR_INTERNAL;
  }
}

// Kaczmarz divisor: proj_diag, and its exact reciprocal when a power of two
template <typename T>
struct KzCoef {
  T proj_diag, recip;
  bool pow2;
};

// Coarse hierarchy kernel (kernels_coarse.cu): one CTA per CW RHS columns
// runs every visit of levels m0..Lc out of shared memory.
// M: storage type of the global fields it reads and writes (forig, f_top,
// u_top); levels on chip and all arithmetic are T.
template <typename T, typename M = T>
struct CoarseArgs {
  int m0 = 0, Lc = 0, m = 0, n_sr = 0;
  int mode = 0;  // 0: coarse FMG steps m0+1..Lc; 1: V-cycle segment below Lc+1
  int CW = 1, B = 1;
  i64 ld = 0;
  i64 W[32] = {}, b[32] = {};
  const M* forig[32] = {};  // mode 0: restricted forcing per level
  const M* f_top = nullptr;  // mode 1: f_{Lc}
  M* u_top = nullptr;        // mode 1: in/out u_{Lc}; mode 0: out
  double omega = 1.0;
  KzCoef<T> kz{};
  int trace = 0;  // debug: per-phase clock printf from CTA 0
  // warp-per-column kernel layout (filled by coarse_warp_layout)
  int lgW[32] = {}, off[32] = {}, slen[32] = {};
  int fields = 0, scratch = 0;
  int nw = 1;  // warps per column (coarse_warp_kernel)
  // CTA kernel: 1 = a shared-memory buffer of 2^Lc x CW cells holds the
  // Kaczmarz-projected copy of an on-chip SR level's input (coarse_smem_bytes
  // extra_cells = 2^Lc); 0 = project just in time inside the chains
  int pj = 0;
  // CTA kernel, whole solve on chip (Lc = m): 1 = the f cascade runs in shared
  // memory from forig[m] (extra 2^(m+1) - 2^m0 cells per column) instead of
  // loading each restricted level from global memory
  int fo = 0;
  // fp32 fields (T = float) with fp64 arithmetic: the CTAs keep their levels
  // and compute in fp64, widening on load and rounding once on store
  int f64_arith = 0;
};
template <typename T> void launch_coarse(const CoarseArgs<T>& a, cudaStream_t s);
template <typename T> size_t coarse_smem_bytes(int m0, int Lc, int CW, int extra_cells = 0);
// one warp per RHS column (kernels_coarse_warp.cu): ns = 1 or 2, linear or nonlinear
template <typename T> size_t coarse_warp_layout(CoarseArgs<T>& a, bool ns2, bool nl);
template <typename T> void launch_coarse_warp(const CoarseArgs<T>& a, bool ns2, bool nl, cudaStream_t s);

// Multi-level restriction (f cascade): p[k] receives level (src_level-1-k)
template <typename T>
struct CascadeDst {
  T* p[6] = {};
  int levels = 0;
};
template <typename T>
void launch_cascade(const T* src, i64 n_src, const CascadeDst<T>& dst, i64 ld, int B, cudaStream_t s);
// fp32 fields, fp64 arithmetic: the pair averages in fp64, each level rounded once
void launch_cascade_f64arith(const float* src, i64 n_src, const CascadeDst<float>& dst, i64 ld,
                             int B, cudaStream_t s);

// ---------------------------------------------------------------------------
// Level-visit descriptor (uniform patch geometry: owned width W, buffer b).
// ---------------------------------------------------------------------------
template <typename T>
struct VisitDesc {
  int src = 0;  // SRC_LOAD / SRC_CORR / SRC_FMG
  bool cr = false, epi = false, write_u = true;
  i64 n = 0, ld = 0;
  int B = 0;
  i64 W = 0, b = 0;
  double omega = 1.0, proj_diag = 0.5;
  const T* u_src = nullptr;  // fine input (LOAD, CORR)
  const T* uH = nullptr;     // coarse input (CORR, FMG, CR target)
  const T* uc = nullptr;     // CR target for LOAD / CORR
  const T* f = nullptr;
  T* u_out = nullptr;
  T* uH_out = nullptr;  // epilogue
  T* fH_out = nullptr;
  T* E = nullptr;    // edge records
  int* cnt = nullptr;  // edge counters
  // explicit patch arrays (optional; SRC_LOAD, no epilogue)
  const i64* olo = nullptr;
  const i64* ohi = nullptr;
  const i64* elo = nullptr;
  const i64* ehi = nullptr;
  i64 P = 0;  // number of patches when arrays are given
  // patch-slab sharding (uniform geometry): patches [p_begin, p_begin + p_count)
  // of the level, pair loads clamped to [qlo, qhi] (the slab and its halo;
  // -1: the whole level).  Edge records of the slab's outer boundaries go to
  // E_out[slot][5][Bpad] (slot 0: left edge, 1: right edge) instead of the
  // in-kernel last-arriver protocol when left_remote / right_remote.
  i64 p_begin = 0, p_count = -1;
  i64 qlo = -1, qhi = -1;
  T* E_out = nullptr;
  bool left_remote = false, right_remote = false;
  // functional output (final up visit): partial sums instead of the field
  const T* fun_w = nullptr;
  T* fun_part = nullptr;  // [P][round_up(B, 32)]
  // fp32 fields with fp64 arithmetic (T = float only): every value widens
  // exactly on load, the visit computes in fp64, stores round once to fp32;
  // E / E_out then hold fp64 records (twice the fp32 workspace)
  bool f64_arith = false;
};

// functional J = scale * sum_p sum_{owned i} w_i u_i (w nullptr: unit weights)
template <typename T>
void launch_functional_field(const T* u, const T* w, i64 n, i64 W, i64 ld, int B, T* part,
                             cudaStream_t s);
template <typename T>
void launch_functional_reduce(const T* part, i64 P, int B, T scale, T* out, cudaStream_t s);

// Complete the owned coarse cell at a shard's slab boundary from the two edge
// records (own outbox slot, neighbour's record received in the inbox).
template <typename T>
void launch_edge_fix(const T* rec_left, const T* rec_right, T* fH, i64 s, i64 nf, i64 ld, int B,
                     int which, cudaStream_t st);

template <typename T>
void launch_visit(const VisitDesc<T>& d, cudaStream_t s);

// Any ns (window staged in a per-chain global scratch).
template <typename T>
struct ScratchDesc {
  i64 n = 0, ld = 0;
  int B = 0;
  i64 W = 0, b = 0;  // uniform geometry when olo == nullptr
  const i64* olo = nullptr;
  const i64* ohi = nullptr;
  const i64* elo = nullptr;
  const i64* ehi = nullptr;
  const i64* soff = nullptr;  // per-patch scratch row offset (arrays mode)
  i64 P = 0;
  i64 ns = 1;
  double omega = 1.0, proj_diag = 0.5;
  const T* u_in = nullptr;
  const T* f = nullptr;
  const T* uc = nullptr;  // non-null => CR
  T* out = nullptr;
  T* scratch = nullptr;
  i64 sld = 0;  // scratch row stride (>= round_up(B, 32))
  bool nonlinear = false;  // Newton-GS for -u'' + u^3 = f
};

template <typename T>
void launch_smooth_scratch(const ScratchDesc<T>& d, cudaStream_t s);

// ns = 2 (V(2,2)) streaming smoother, uniform geometry: forward chain with the
// visit prologue, window spilled to scratch, backward chain from the spill.
template <typename T>
struct Ns2Desc {
  int src = 0;  // SRC_LOAD / SRC_CORR / SRC_FMG
  bool cr = false, nonlinear = false;
  i64 n = 0, ld = 0;
  int B = 0;
  i64 W = 0, b = 0;
  double omega = 1.0, proj_diag = 0.5;
  const T* u_src = nullptr;
  const T* uH = nullptr;
  const T* uc = nullptr;
  const T* f = nullptr;
  T* u_out = nullptr;
  T* scratch = nullptr;  // (n / W) * (W + 2b + 2) rows of sld
  i64 sld = 0;
  // fused restriction + tau (T / D visits; nonlinear tau when nonlinear)
  bool epi = false, write_u = true;
  T* uH_out = nullptr;
  T* fH_out = nullptr;
  T* E = nullptr;
  int* cnt = nullptr;
};

template <typename T>
void launch_smooth_ns2(const Ns2Desc<T>& d, cudaStream_t s);
inline i64 scratch_rows_uniform(i64 n, i64 W, i64 b) { return (n / W) * (W + 2 * b + 2); }

// Stencil / level operators ([n][ld] layout, B active columns).
template <typename T> void launch_apply_operator(const T* u, T* out, i64 n, i64 ld, int B, cudaStream_t s);
template <typename T> void launch_restrict(const T* u, T* out, i64 nf, i64 ld, int B, cudaStream_t s);
template <typename T> void launch_prolong_correction(const T* c, T* out, i64 nc, i64 ld, int B, cudaStream_t s);
template <typename T> void launch_prolong_fmg(const T* c, T* out, i64 nc, i64 ld, int B, cudaStream_t s);
// mode 0: tau only; 1: coarse_rhs; 2: restrict + coarse_rhs (uH_out, fH_out);
// nl: tau of the nonlinear operator N(u) = L u + u^3
template <typename T> void launch_restrict_tau(const T* u, const T* f, T* uH_out, T* fH_out, i64 nf, i64 ld, int B, int mode, cudaStream_t s, bool nl = false);
// Newton solve of L u + u^3 = f on the coarsest level (n <= 64)
template <typename T> void launch_direct_solve_nl(const T* f, T* u, i64 n, i64 ld, int B, cudaStream_t s);
template <typename T> void launch_fas_correct(const T* u, const T* uH, T* out, i64 nf, i64 ld, int B, cudaStream_t s);
template <typename T> void launch_direct_solve(const T* f, T* u, i64 n, i64 ld, int B, cudaStream_t s, T* workspace = nullptr);
// peer-memory transport of the sharded plan (kernels_p2p.cu): per-rank
// counter words and one step's pulls
enum { P2P_READY = 0, P2P_FIXED = 1, P2P_DONE = 2, P2P_EPOCH = 3, P2P_ERR = 4, P2P_NWORDS = 8 };
constexpr int P2P_MAXE = 40, P2P_MAXW = 16;
// A slab-edge fix-up folded into the exchange kernel: coarse cells s/2-1, s/2
// of f_H from the left (L) and right (R) 5-value edge records (k_edge_fix).
struct P2pFix {
  const void* L;
  const void* R;
  void* fH;
  i64 s, nf, ld, ldE;
  int B;
};
struct P2pCopy {
  int n = 0, nwait = 0, signal = -1;  // signal: counter word to publish first (-1: none)
  int nfix = 0;
  unsigned long long nstep = 0, step = 0, timeout_ns = 0;
  const unsigned long long* wait[P2P_MAXW];
  const void* src[P2P_MAXE];
  void* dst[P2P_MAXE];
  unsigned long long bytes[P2P_MAXE];
  unsigned char cta0[P2P_MAXE];  // copied by CTA 0 alone (fix-up inputs and outputs)
  P2pFix fix[2];
};
void launch_p2p_epoch(unsigned long long* flags, cudaStream_t s);
template <typename T>
void launch_p2p_wait_copy(const P2pCopy& c, unsigned long long* flags, cudaStream_t s);
template <typename T> void launch_banded_lu_solve(const T* f, T* u, i64 n, i64 ld, int B, T* workspace, int* bad, cudaStream_t s);
template <typename T> void launch_gs_sweep(T* u, const T* f, i64 n, i64 ld, int B, double inv_h2, i64 start, i64 stop, bool forward, double omega, cudaStream_t s);
template <typename T> void launch_kaczmarz_sweep(T* u, const T* uc, i64 n, i64 ld, int B, i64 start, i64 stop, double proj_diag, cudaStream_t s);
template <typename T> void launch_fourier_rhs(const double* coef, int K, i64 n, i64 ld, int B, T* f, T* uex, cudaStream_t s);
void launch_manufactured(i64 n, i64 K, double* f, double* uex, cudaStream_t s);
template <typename T> void launch_div_check(const T* x, const T* J, T* q, i64 n, unsigned long long* bad, cudaStream_t s);
template <typename T> void launch_nonlinear_rhs(const double* scale, i64 n, i64 ld, int B, T* f, T* uex, cudaStream_t s);

}  // namespace fmgsr
