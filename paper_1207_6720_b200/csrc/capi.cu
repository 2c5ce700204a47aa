// capi.cu -- extern "C" boundary of libfmgsr_cuda.so (include/fmgsr_cuda.h)
// and the native FMG-FAS(-SR) solve plan.
//
// The plan is the B200-side replacement of the reference driver
// (cycles.py:95-222): it owns the per-level device workspace, derives the
// level-visit schedule once, emits one fused kernel per level visit where
// the visit qualifies (ns = 1, owned width >= 4 for visits that restrict),
// and captures the whole cycle into a CUDA graph that is replayed per solve.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <mutex>
#include <map>
#include <memory>
#include <tuple>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fmgsr_cuda.h"
#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

int smem_optin(const void* kf) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> granted;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "smem opt-in device");
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, kf);
  auto it = granted.find(key);
  if (it != granted.end()) return it->second;
  int optin = 0;
  check_cuda(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
             "smem opt-in limit");
  cudaFuncAttributes fa;
  check_cuda(cudaFuncGetAttributes(&fa, kf), "kernel attributes");
  const int g = optin - (int)fa.sharedSizeBytes;
  check_cuda(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, g),
             "smem opt-in");
  granted.emplace(key, g);
  return g;
}

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
void clear_last_error() { g_last_error.clear(); }

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static void check_field(i64 n, i64 B, i64 ld, const char* what) {
  require(n >= 1, std::string(what) + ": empty level");
  require(B >= 1 && B <= (i64)1 << 30, std::string(what) + ": B out of range");
  require(ld >= B, std::string(what) + ": ld < B");
}

// ===========================================================================
// Plan
// ===========================================================================
enum VisitKind { VK_TOP = 0, VK_DOWN = 1, VK_UP = 2, VK_DIRECT = 3, VK_CASCADE = 4, VK_COARSE = 5 };

struct LevelGeo {
  i64 W, b;
};

static LevelGeo level_geometry(i64 n, int mode, i64 P, i64 b) {
  // reference mesh.py:102-136; mode 2 = generalised P-patch rule
  if (mode == 1) return {n, 0};
  if (mode == 0) return {2, b};
  i64 w = n / P;
  return {w < 2 ? 2 : w, b};
}

// ---------------------------------------------------------------------------
// Patch-slab sharding transport.  A sharded plan owns one contiguous slab of
// patches on every level above the replication cutoff Lr; after each visit
// it exchanges halo rows and slab-edge tau records with its two neighbours
// and, at Lr, all-gathers the restricted level so everything below runs
// replicated.  Transfers are described, not performed, by the plan:
// ShardGroup (virtual shards on one device) turns them into device copies,
// NcclComm (one shard per GPU) into grouped ncclSend / ncclRecv / ncclAllGather.
// ---------------------------------------------------------------------------
struct Xfer {
  int peer;
  bool send;
  void* ptr;
  size_t bytes;
  int tag;
  int lvl;  // level of the array moved (-1: tau edge record)
};
struct Gather {
  char* base;    // the full (replicated) array
  size_t chunk;  // bytes owned by each shard, shard k at base + k * chunk
};

struct NcclApi;  // dlopen'ed libnccl (only when a multi-GPU sharded plan is built)

struct PlanBase {
  fmgsr_plan_desc d{};
  virtual ~PlanBase() {}
  virtual void solve(const void* in, void* out, cudaStream_t s) = 0;
  // durations (ms) of the finest top / up visits of the last completed solve; -1 if none
  virtual void probe_ms(float* top, float* up) { *top = *up = -1.0f; }
  virtual void solve_timed(const void* in, void* out, cudaStream_t s, float* ms, int32_t* lvl,
                           int32_t* kind, i64 cap, i64* nv) = 0;
  virtual void info(fmgsr_plan_info* inf) = 0;
  virtual void solve_host(const void* h_in, void* h_out, i64 ld_host, i64 chunks,
                          cudaStream_t s, int flags) = 0;
  virtual void solve_functional(const void* in, const void* w, void* out, cudaStream_t s) = 0;
  virtual void set_debug(int flags) = 0;
  virtual i64 check_guards() = 0;
  // peer-memory transport of a sharded plan (fmgsr_shard_plan_create_p2p)
  virtual size_t p2p_export(void* buf, size_t cap) {
    (void)buf, (void)cap;
    throw Error(ERR_ARG, "not a peer-memory shard plan");
  }
  virtual void p2p_import(const char* all, size_t per_rank) {
    (void)all, (void)per_rank;
    throw Error(ERR_ARG, "not a peer-memory shard plan");
  }
  virtual int p2p_status() { throw Error(ERR_ARG, "not a peer-memory shard plan"); }
  // a sharded plan's own finest forcing buffer (slab rows, halo rows around them)
  virtual void* forcing_slab(i64* rows) {
    (void)rows;
    throw Error(ERR_ARG, "not a sharded plan");
  }
};

template <typename T>
struct Plan : PlanBase {
  struct Level {
    i64 n = 0, W = 0, b = 0;
    T* u[2] = {nullptr, nullptr};
    void* ub[2] = {nullptr, nullptr};  // allocation bases of u[0], u[1] (debug poisoning)
    size_t ubytes = 0;
    int cur = 0;
    T* f = nullptr;
    T* E = nullptr;
    int* cnt = nullptr;
  };
  std::vector<Level> lv;
  T* tmp = nullptr;
  T* scratch = nullptr;
  i64 sld = 0;
  int* cnt_all = nullptr;
  size_t cnt_bytes = 0;
  std::vector<void*> allocs;       // raw cudaMalloc pointers
  std::vector<void*> alloc_user;   // what alloc() returned (after the front guard)
  std::vector<size_t> alloc_sizes;
  // Debug aids in place of compute-sanitizer (closed on this pool):
  //  guards (FMGSR_GUARDS=1 at plan creation): every workspace array sits
  //    between two 4 KiB guard zones filled with 0x5A; check_guards() counts
  //    changed guard bytes -- an out-of-bounds write detector;
  //  FMGSR_DEBUG_POISON (fmgsr_plan_set_debug): every solve first fills the
  //    level fields, edge records and scratch with NaN (uninitialised reads
  //    would surface in the result), and after each FMG step fills the SR
  //    levels below it with NaN -- the reference's debug_sr (cycles.py:161-165,
  //    209-212): the only field a step may read from the previous one is the
  //    previous finest level.
  static constexpr size_t GUARD = 4096;
  bool guards = false;
  int debug = 0;
  size_t n_field_allocs = 0;  i64 ws_bytes = 0;
  cudaStream_t cap = nullptr;
  std::map<std::pair<const void*, void*>, cudaGraphExec_t> graphs;
  // probe events around the finest-level top and up visits, recorded by every
  // solve (as event-record nodes inside the captured graphs): after a solve
  // completes they hold that solve's durations of T_m and U_m
  cudaEvent_t probe_ev[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int probe_open = -1;
  // per-solve bookkeeping (filled by enqueue)
  i64 n_launch = 0, n_visit = 0;
  // timing hooks
  std::vector<cudaEvent_t> ev;
  std::vector<int32_t> ev_lvl, ev_kind;
  bool timing = false;
  // coarse hierarchy kernel: levels m0..Lc on chip, CW RHS columns per CTA
  bool use_coarse = false, coarse_warp = true;
  // whole solve on chip (Lc = m): every level, the finest included, in one
  // coarse launch after the f cascade
  bool whole = false;
  int Lc = 0, CW = 1;
  int CNW = 1;  // warp kernel: warps per column (one chain per thread on level Lc)
  int coarse_trace = 0;
  // patch-slab sharding: levels > Lr are split into S slabs, this is slab srank;
  // slab arrays carry H halo rows per side and are addressed through
  // "virtual global" pointers (global row g at base + (g - c0 + H) * ld)
  int S = 1, srank = 0, Lr = 1 << 30;
  i64 H = 0;
  T* fm = nullptr;  // sharded finest forcing (slab + halo)
  T* fm_base = nullptr;  // its allocation
  // the caller may fill the plan's own forcing slab (forcing_slab()) and pass
  // it to solve: then ST_LOADF has nothing to copy
  bool forcing_in_place(const T* forcing) const {
    return S > 1 && forcing == fm + c0(d.m) * d.ld;
  }
  void* forcing_slab(i64* rows) override {
    require(S > 1 && fm, "forcing_slab: not a sharded plan");
    if (rows) *rows = c1(d.m) - c0(d.m);
    return fm + c0(d.m) * d.ld;
  }
  std::vector<T*> ob, ib;  // per-level edge-record outbox / inbox (2 slots x 5 x Bp)
  bool sharded(int l) const { return S > 1 && l > Lr; }
  i64 c0(int l) const { return (lv[l].n / S) * srank; }
  i64 c1(int l) const { return (lv[l].n / S) * (srank + 1); }

  bool is_sr(int l) const { return l > d.m - d.n_sr; }

  // Levels whose visits carry the fused restriction + tau epilogue (edge
  // records and counters allocated): owned width >= 4, or width 2 where the
  // short-patch group kernel serves the down visits (a group owns >= 4 cells).
  bool group_w2(const Level& L) const {
    return d.fused && d.ns == 1 && !d.nonlinear && !mixed && L.W == 2 && L.n >= 8 &&
           L.b <= 32 && group_visit_enabled();  // try_group_visit's own limits
  }
  bool epi_level(const Level& L) const { return L.W >= 4 || group_w2(L); }

  // Dry plans (fmgsr_shard_schedule) run the host logic only -- geometry,
  // cutoffs, the step list and its level ping-pong state -- with every device
  // call skipped and fake addresses, so the communication schedule can be
  // exported and checked without a GPU.  The B200's attributes stand in for
  // the device's.
  bool dry = false;
  uintptr_t dry_next = (uintptr_t)1 << 44;
  // local shard plans (fmgsr_shard_plan_create_local): no transport at all,
  // for timing one shard's work on one GPU (results are not a solve)
  bool local = false;
  int devattr(cudaDeviceAttr a, int b200) const {
    if (dry) return b200;
    int dev = 0, v = 0;
    check_cuda(cudaGetDevice(&dev), "device");
    check_cuda(cudaDeviceGetAttribute(&v, a, dev), "device attribute");
    return v;
  }
#define FMGSR_PLAN_FWD(NAME) \
  template <class... A> void NAME(A&&... a) { if (!dry) fmgsr::NAME(std::forward<A>(a)...); }
  // fp32 fields with fp64 arithmetic (dtype 2, T = float): every kernel
  // widens on load, computes in fp64 and rounds once per stored value; edge
  // records and the on-chip coarse levels are fp64
  bool mixed = false;
  size_t esz() const { return mixed ? sizeof(double) : sizeof(T); }  // arithmetic element
  void launch_visit(VisitDesc<T> v, cudaStream_t s) {
    if (dry) return;
    v.f64_arith = mixed;
    fmgsr::launch_visit(v, s);
  }
  void launch_cascade(const T* src, i64 n_src, const CascadeDst<T>& dst, i64 ld, int B,
                      cudaStream_t s) {
    if (dry) return;
    if constexpr (std::is_same<T, float>::value) {
      if (mixed) {
        launch_cascade_f64arith(src, n_src, dst, ld, B, s);
        return;
      }
    }
    fmgsr::launch_cascade(src, n_src, dst, ld, B, s);
  }
  FMGSR_PLAN_FWD(launch_restrict_tau)
  FMGSR_PLAN_FWD(launch_prolong_fmg)
  FMGSR_PLAN_FWD(launch_fas_correct)
  FMGSR_PLAN_FWD(launch_direct_solve)
  FMGSR_PLAN_FWD(launch_direct_solve_nl)
  FMGSR_PLAN_FWD(launch_coarse)
  FMGSR_PLAN_FWD(launch_coarse_warp)
  FMGSR_PLAN_FWD(launch_smooth_ns2)
  FMGSR_PLAN_FWD(launch_smooth_scratch)
  FMGSR_PLAN_FWD(launch_edge_fix)
  FMGSR_PLAN_FWD(launch_functional_field)
  FMGSR_PLAN_FWD(launch_functional_reduce)
#undef FMGSR_PLAN_FWD

  std::vector<std::pair<uintptr_t, size_t>> dry_allocs;  // dry plans: fake base, bytes
  size_t n_init_allocs = 0;  // allocations made by init() (the exported workspace)
  T* alloc(size_t bytes) {
    if (dry) {
      const uintptr_t p = dry_next;
      dry_next += (bytes + 255) / 256 * 256 + 4096;
      ws_bytes += (i64)bytes;
      dry_allocs.push_back({p, bytes ? bytes : 16});
      return (T*)p;
    }
    void* p = nullptr;
    const size_t ub = bytes ? bytes : 16, g = guards ? GUARD : 0;
    check_cuda(cudaMalloc(&p, ub + 2 * g), "plan workspace cudaMalloc");
    allocs.push_back(p);
    if (g) check_cuda(cudaMemset(p, 0x5A, ub + 2 * g), "guard fill");
    p = (char*)p + g;
    alloc_user.push_back(p);
    alloc_sizes.push_back(ub);
    ws_bytes += (i64)bytes;
    return (T*)p;
  }

  // A constructor that throws never runs the destructor: release() frees
  // whatever was created so far (also called by the destructor).
  explicit Plan(const fmgsr_plan_desc& desc, int shards = 1, int shard = 0, bool dry_ = false,
                bool local_ = false) {
    dry = dry_;
    local = local_;
    const char* ge = getenv("FMGSR_GUARDS");
    guards = !dry && ge && ge[0] == '1';
    try {
      init(desc, shards, shard);
    } catch (...) {
      release();
      throw;
    }
  }
  void init(const fmgsr_plan_desc& desc, int shards, int shard) {
    d = desc;
    S = shards;
    srank = shard;
    mixed = d.dtype == 2;
    if (mixed)
      require(d.fused && d.ns == 1 && !d.nonlinear && d.coarse != 0 && S == 1,
              "fp64 arithmetic on fp32 fields: the fused ns = 1 linear plan with the on-chip "
              "coarse levels, unsharded");
    const int m0 = d.m0, m = d.m;
    const i64 ld = d.ld, Bp = ((d.B + 31) / 32) * 32;
    const int nrg = (int)(Bp / 32);
    lv.resize(m + 1);
    i64 tmp_rows = 0, scratch_rows = 0, cnt_total = 0;
    for (int l = m0; l <= m; l++) {
      Level& L = lv[l];
      L.n = (i64)1 << l;
      LevelGeo g = level_geometry(L.n, d.geom_mode, d.P, d.b);
      L.W = g.W;
      L.b = g.b;
      require(L.n % L.W == 0, "plan: owned width does not divide the level");
      if (l > m0 && (d.ns >= 2 || d.nonlinear)) {
        i64 rows = scratch_rows_uniform(L.n, L.W, L.b);
        if (rows > scratch_rows) scratch_rows = rows;
      }
      if (l > m0) tmp_rows = L.n > tmp_rows ? L.n : tmp_rows;
      if (l > m0 && epi_level(L)) cnt_total += (L.n / L.W + 1) * nrg;
    }
    // Coarse cutoff: about 128 CTAs of CW columns; the deepest level whose
    // three fields per level (two u, f) for CW columns fit in ~200 KB.
    // Two coarse kernels: one warp per RHS column (default; ns 1 or 2, linear or
    // nonlinear) or one CTA per CW columns (FMGSR_COARSE=cta; ns = 1 linear).
    // The CTA kernel is faster where it applies (measured: config 2 3.30 vs
    // 3.70 ms); the warp kernel carries ns = 2 and the nonlinear smoother.
    const char* ck = getenv("FMGSR_COARSE");
    coarse_warp = !mixed && ((d.ns != 1 || d.nonlinear) || (ck && std::string(ck) == "warp"));
    use_coarse = d.fused && d.coarse != 0 && (d.ns == 1 || d.ns == 2) && d.m - d.m0 >= 2;
    const char* tr = getenv("FMGSR_COARSE_TRACE");
    coarse_trace = (tr && tr[0] == '1') ? 1 : 0;
    if (use_coarse && coarse_warp) {
      // deepest Lc whose per-warp slice fits and keeps all B warps in one wave
      CW = 1;
      Lc = m0;
      const int smsm = devattr(cudaDevAttrMaxSharedMemoryPerMultiprocessor, 233472);
      const int nsm = devattr(cudaDevAttrMultiProcessorCount, 148);
      // warps per column: one chain per thread on the deepest level (a
      // thread's serial work grows with P_l / (32 NW)), at most 8 warps
      auto nw_for = [&](int lc) {
        int nw = 1;
        while (nw < 8 && 32 * nw < lv[lc].n / lv[lc].W) nw *= 2;
        return nw;
      };
      int max_nw = 8;
      if (const char* e = getenv("FMGSR_COARSE_NW")) max_nw = atoi(e);
      auto fits = [&](int lc) {
        CoarseArgs<T> t;
        t.m0 = m0;
        t.Lc = lc;
        t.nw = nw_for(lc);
        if (t.nw > max_nw || 32 * t.nw < lv[lc].n / lv[lc].W) return false;
        for (int l = m0; l <= lc; l++) {
          t.W[l] = lv[l].W;
          t.b[l] = lv[l].b;
        }
        const size_t bytes = coarse_warp_layout(t, d.ns == 2, d.nonlinear != 0);
        if (bytes > 227 * 1024) return false;
        i64 per_sm = (i64)smsm / (i64)(bytes + 1024);
        if (per_sm > 64 / t.nw) per_sm = 64 / t.nw;
        return per_sm >= 1 && per_sm * nsm >= d.B;
      };
      while (Lc + 1 <= m - 1 && fits(Lc + 1)) Lc++;
      {  // the coarsest level itself must fit one CTA's shared memory
        CoarseArgs<T> t;
        t.m0 = m0;
        t.Lc = m0;
        t.nw = nw_for(m0);
        t.W[m0] = lv[m0].W;
        t.b[m0] = lv[m0].b;
        if (coarse_warp_layout(t, d.ns == 2, d.nonlinear != 0) > 227 * 1024) use_coarse = false;
      }
      int want = d.coarse;
      if (want < 0)
        if (const char* e = getenv("FMGSR_COARSE_LC")) want = atoi(e) + 1;
      if (want > 0 && want - 1 >= m0 && want - 1 < Lc) Lc = want - 1;
      CNW = nw_for(Lc);
    } else if (use_coarse) {
      i64 cw = 1;
      // ~128 CTAs (one wave on 148 SMs); measured best against 256 / 512
      i64 target = 128;
      if (const char* e = getenv("FMGSR_COARSE_CTAS")) target = atoll(e);
      while (cw * 2 <= 32 && cw * 2 * target <= d.B) cw *= 2;
      if (const char* e = getenv("FMGSR_COARSE_CW")) cw = atoll(e);  // A/B experiments
      CW = (int)cw;
      Lc = m0;
      // an on-chip SR level adds a projected-copy buffer of 2^Lc cells per column
      auto smem_at = [&](int lc) {
        return mixed ? coarse_smem_bytes<double>(m0, lc, CW, lc > m - d.n_sr ? 1 << lc : 0)
                     : coarse_smem_bytes<T>(m0, lc, CW, lc > m - d.n_sr ? 1 << lc : 0);
      };
      // the coarsest level itself must fit: fewer columns per CTA, else no coarse kernel
      while (CW > 1 && smem_at(m0) > 200 * 1024) CW /= 2;
      if (smem_at(m0) > 200 * 1024) use_coarse = false;
      while (Lc + 1 <= m - 1 && smem_at(Lc + 1) <= 200 * 1024) Lc++;
      int want = d.coarse;
      if (want < 0)
        if (const char* e = getenv("FMGSR_COARSE_LC")) want = atoi(e) + 1;
      if (want > 0 && want - 1 >= m0 && want - 1 < Lc) Lc = want - 1;
      // Whole solve on chip when every level fits and the column groups fill at
      // most one wave (small batches, e.g. config 1: one RHS, N = 2^10): the
      // finest visits then run from shared memory too and a solve is two
      // launches (auto, or coarse = m + 1; FMGSR_COARSE_WHOLE=0 disables).
      const char* we = getenv("FMGSR_COARSE_WHOLE");
      const bool allow = !(we && we[0] == '0') && !mixed;
      const int nsm = devattr(cudaDevAttrMultiProcessorCount, 148);
      const bool fits = coarse_smem_bytes<T>(m0, m, CW, (m > m - d.n_sr ? 1 << m : 0) +
                                                           (1 << (m + 1)) - (1 << m0)) <= 200 * 1024 &&
                        (d.B + CW - 1) / CW <= nsm;
      if (S == 1 && !mixed && fits && ((want < 0 && allow) || want == m + 1)) {
        whole = true;
        Lc = m;
      }
    }
    if (mixed) {
      require(use_coarse, "fp64 arithmetic on fp32 fields needs the on-chip coarse levels");
      for (int l = Lc + 1; l <= m; l++)
        require(lv[l].W >= 4, "fp64 arithmetic on fp32 fields: every level above the on-chip "
                              "cutoff needs owned width >= 4 (the fused restriction)");
    }
    if (S > 1) {
      require(use_coarse, "sharding needs the on-chip coarse levels (coarse != 0)");
      plan_shards(Bp);
      finish_shards();
    }
    ob.assign(m + 1, nullptr);
    ib.assign(m + 1, nullptr);
    for (int l = m0; l <= m; l++) {
      Level& L = lv[l];
      if (sharded(l)) {
        // slab + halo; pointers stored shifted to virtual global rows
        const i64 rows = L.n / S + 2 * H, shift = (H - c0(l)) * ld;
        size_t fb = (size_t)rows * ld * sizeof(T);
        L.u[0] = alloc(fb) + shift;
        L.u[1] = alloc(fb) + shift;
        L.ub[0] = L.u[0] - shift;
        L.ub[1] = L.u[1] - shift;
        L.ubytes = fb;
        if (l < m) L.f = alloc(fb) + shift;
        else fm = (fm_base = alloc(fb)) + shift;
        ob[l] = alloc((size_t)10 * Bp * sizeof(T));
        ib[l] = alloc((size_t)10 * Bp * sizeof(T));
      } else {
        size_t fb = (size_t)L.n * ld * sizeof(T);
        L.u[0] = alloc(fb);
        L.u[1] = alloc(fb);
        L.ub[0] = L.u[0];
        L.ub[1] = L.u[1];
        L.ubytes = fb;
        if (l < m) L.f = alloc(fb);
      }
      if (l > m0 && epi_level(L)) L.E = alloc((size_t)(L.n / L.W + 1) * 10 * Bp * esz());
    }
    tmp = alloc((size_t)tmp_rows * ld * sizeof(T));
    if (!dry)
      for (auto& pe : probe_ev)
        for (auto& e : pe) check_cuda(cudaEventCreate(&e), "probe event");
    if (scratch_rows) {
      sld = Bp;
      scratch = alloc((size_t)scratch_rows * sld * sizeof(T));
    }
    n_field_allocs = allocs.size();  // everything so far is rewritten before it is read
    cnt_bytes = (size_t)cnt_total * sizeof(int);
    cnt_all = (int*)alloc(cnt_bytes);
    if (!dry) check_cuda(cudaMemset(cnt_all, 0, cnt_bytes ? cnt_bytes : 16), "plan memset");
    if (local)  // no halo ever arrives: keep the never-written rows finite
      for (size_t k = 0; k < allocs.size(); k++)
        check_cuda(cudaMemset(alloc_user[k], 0, alloc_sizes[k]), "plan memset");
    i64 off = 0;
    for (int l = m0 + 1; l <= m; l++) {
      Level& L = lv[l];
      if (epi_level(L)) {
        L.cnt = cnt_all + off;
        off += (L.n / L.W + 1) * nrg;
      }
    }
    n_init_allocs = dry ? dry_allocs.size() : allocs.size();
    if (!dry) check_cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "plan stream");
  }

  // Replication cutoff: every level above Lr must split into S slabs of whole
  // patches with owned width >= 4 (fused restriction epilogue) and room for
  // the halo; Lr >= Lc (the on-chip levels are replicated anyway).
  void plan_shards(i64 Bp) {
    (void)Bp;
    require(d.fused && d.ns == 1 && !d.nonlinear && d.coarse != 0,
            "sharding needs the fused ns = 1 linear path");
    require(S >= 2 && is_pow2(S) && srank >= 0 && srank < S, "bad shard count / index");
    H = d.b + 8;
    H += H & 1;
    auto ok = [&](int l) {
      const Level& L = lv[l];
      const i64 slab = L.n / S;
      return L.n % S == 0 && slab % L.W == 0 && L.W >= 4 && slab >= 2 * H && slab >= 64;
    };
    require(ok(d.m), "sharding: the finest level cannot be split into S patch slabs");
    int l = d.m;
    while (l - 1 > d.m0 && ok(l - 1)) l--;
    Lr = l - 1;
  }
  void finish_shards() {  // after the coarse cutoff is known
    if (S > 1 && Lr < Lc) {
      // levels Lr+1..Lc would be both sharded and on chip: shard only above Lc
      Lr = Lc;
      require(Lr < d.m, "sharding: nothing left above the coarse cutoff");
    }
  }
  void shard_desc(VisitDesc<T>& v, int l) const {
    if (!sharded(l)) return;
    const Level& L = lv[l];
    v.p_begin = c0(l) / L.W;
    v.p_count = (c1(l) - c0(l)) / L.W;
    const i64 lo = c0(l) - H, hi = c1(l) + H;  // rows in memory
    v.qlo = lo < 0 ? 0 : lo / 2;
    v.qhi = (hi > L.n ? L.n : hi) / 2 - 1;
    if (v.epi) {
      v.E_out = ob[l];
      v.left_remote = c0(l) > 0;
      v.right_remote = c1(l) < L.n;
    }
  }

  ~Plan() override { release(); }
  void release() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
    for (auto& kv : fgraphs) cudaGraphExecDestroy(kv.second);
    fgraphs.clear();
    for (auto& pe : probe_ev)
      for (auto& e : pe)
        if (e) cudaEventDestroy(e), e = nullptr;
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    for (auto e : hev) cudaEventDestroy(e);
    hev.clear();
    if (cap) cudaStreamDestroy(cap), cap = nullptr;
    if (s_in) cudaStreamDestroy(s_in), s_in = nullptr;
    if (s_out) cudaStreamDestroy(s_out), s_out = nullptr;
    if (ncomm && nccl && nccl->commDestroy) nccl->commDestroy(ncomm);
    ncomm = nullptr;
    if (p2p) {
      for (void* q : p2p->opened) cudaIpcCloseMemHandle(q);
      if (p2p->flags) cudaFree(p2p->flags);
      delete p2p;
      p2p = nullptr;
    }
    if (!dry)
      for (void* p : allocs) cudaFree(p);
    allocs.clear();
    alloc_user.clear();
    alloc_sizes.clear();
  }

  // ---- host-buffer solve: chunks of B columns pipelined over PCIe ---------------
  // Host arrays are [N][ld_host] with chunks * B columns.  Chunk i is copied
  // (one cudaMemcpy2DAsync) into device buffer set i % 2 on s_in, solved on the
  // caller's stream by the plan's graph for that buffer set, and copied back on
  // s_out, so H2D of chunk i+1, the solve of chunk i and D2H of chunk i-1
  // overlap.  The two buffer sets are allocated on first use.
  cudaStream_t s_in = nullptr, s_out = nullptr;
  T* hbuf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [set][forcing, solution]
  std::vector<cudaEvent_t> hev;  // in_done[2], solved[2], out_done[2]

  bool host_primed = false;  // staging events carry the previous host solve's state
  void solve_host(const void* h_in, void* h_out, i64 ld_host, i64 chunks,
                  cudaStream_t s, int flags) override {
    const i64 N = (i64)1 << d.m, B = d.B;
    require(d.ld == B, "solve_host: the plan must be built with ld == B (one chunk)");
    require(chunks >= 1 && ld_host >= chunks * B, "solve_host: ld_host < chunks * B");
    if (!s_in) {
      check_cuda(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking), "h2d stream");
      check_cuda(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking), "d2h stream");
      for (int k = 0; k < 2; k++)
        for (int j = 0; j < 2; j++) hbuf[k][j] = alloc((size_t)N * B * sizeof(T));
      hev.resize(6);
      for (auto& e : hev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ev");
    }
    cudaEvent_t *in_done = &hev[0], *solved = &hev[2], *out_done = &hev[4];
    const size_t row = (size_t)B * sizeof(T), pitch = (size_t)ld_host * sizeof(T);
    // Strict (default): the H2D copies are ordered after prior work on `stream`.
    // FMGSR_HOST_INPUTS_READY: the host inputs are ready at call time, so the
    // H2D copies only wait for the staging buffers of the previous host solve
    // to be released -- consecutive calls stream (this call's H2D overlaps the
    // previous call's D2H tail).  The solves stay on `stream` either way.
    if (!(flags & FMGSR_HOST_INPUTS_READY) || !host_primed) {
      for (int k = 0; k < 2; k++) {
        check_cuda(cudaEventRecord(solved[k], s), "ev");
        check_cuda(cudaEventRecord(out_done[k], s), "ev");
      }
    }
    host_primed = true;
    for (i64 i = 0; i < chunks; i++) {
      const int k = (int)(i & 1);
      const char* src = (const char*)h_in + i * row;
      char* dst = (char*)h_out + i * row;
      // H2D of chunk i once the solve of chunk i-2 no longer reads forcing set k
      check_cuda(cudaStreamWaitEvent(s_in, solved[k], 0), "wait");
      check_cuda(cudaMemcpy2DAsync(hbuf[k][0], row, src, pitch, row, N, cudaMemcpyHostToDevice,
                                   s_in),
                 "h2d");
      check_cuda(cudaEventRecord(in_done[k], s_in), "ev");
      // solve once the input landed and the D2H of chunk i-2 drained solution set k
      check_cuda(cudaStreamWaitEvent(s, in_done[k], 0), "wait");
      check_cuda(cudaStreamWaitEvent(s, out_done[k], 0), "wait");
      solve(hbuf[k][0], hbuf[k][1], s);
      check_cuda(cudaEventRecord(solved[k], s), "ev");
      check_cuda(cudaStreamWaitEvent(s_out, solved[k], 0), "wait");
      check_cuda(cudaMemcpy2DAsync(dst, pitch, hbuf[k][1], row, row, N, cudaMemcpyDeviceToHost,
                                   s_out),
                 "d2h");
      check_cuda(cudaEventRecord(out_done[k], s_out), "ev");
    }
    for (int k = 0; k < 2; k++) check_cuda(cudaStreamWaitEvent(s, out_done[k], 0), "wait");
  }

  // ---- visit emitters ---------------------------------------------------
  // inside a stream capture an event record becomes a graph node only with
  // cudaEventRecordExternal (a plain record is a capture-internal dependency)
  void probe_record(cudaEvent_t e, cudaStream_t s) const {
    if (dry) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    check_cuda(cudaStreamIsCapturing(s, &st), "capture status");
    if (st == cudaStreamCaptureStatusActive)
      check_cuda(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal), "probe record");
    else
      check_cuda(cudaEventRecord(e, s), "probe record");
  }
  // NVTX range per level visit ("T_24", "D_23", "U_24", "C_12", "F_24", "X_3"),
  // so ncu --nvtx --nvtx-include "U_20/" picks one visit of an op-by-op solve
  void nvtx_push(int lvl, int kind) const {
    if (dry) return;
    static const char kc[] = {'T', 'D', 'U', 'X', 'F', 'C'};
    char name[16];
    snprintf(name, sizeof name, "%c_%d", kc[kind], lvl);
    nvtxRangePushA(name);
  }
  void mark_begin(cudaStream_t s, int lvl, int kind) {
    nvtx_push(lvl, kind);
    n_visit++;
    probe_open = -1;
    if (lvl == d.m && (kind == VK_TOP || kind == VK_UP) && probe_ev[0][0] && !dry) {
      probe_open = kind == VK_TOP ? 0 : 1;
      probe_record(probe_ev[probe_open][0], s);
    }
    if (!timing) return;
    cudaEvent_t a;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventRecord(a, s), "event record");
    ev.push_back(a);
    ev_lvl.push_back(lvl);
    ev_kind.push_back(kind);
  }
  void mark_end(cudaStream_t s) {
    if (!dry) nvtxRangePop();
    if (probe_open >= 0) {
      probe_record(probe_ev[probe_open][1], s);
      probe_open = -1;
    }
    if (!timing) return;
    cudaEvent_t b;
    check_cuda(cudaEventCreate(&b), "event");
    check_cuda(cudaEventRecord(b, s), "event record");
    ev.push_back(b);
  }

  bool fused_restrict_ok(const Level& L) const {
    return d.fused && d.ns == 1 && L.W >= 4 && !d.nonlinear;
  }
  // fused prologue + ns = 1 chain (linear smoother only)
  bool fused_chain_ok() const { return d.fused && d.ns == 1 && !d.nonlinear; }

  // V(2,2) streaming smoother with the visit prologue fused (kernels_ns2.cu)
  bool ns2_ok(const Level& L) const { return d.fused && d.ns == 2 && L.n >= 8; }
  void smooth_ns2(int l, int src, const T* u_src, const T* uH, bool cr, const T* f, T* out,
                  cudaStream_t s, const Ns2Desc<T>* epi = nullptr) {
    const Level& L = lv[l];
    Ns2Desc<T> c;
    if (epi) c = *epi;
    c.src = src;
    c.cr = cr;
    c.nonlinear = d.nonlinear != 0;
    c.n = L.n;
    c.ld = d.ld;
    c.B = (int)d.B;
    c.W = L.W;
    c.b = L.b;
    c.omega = d.omega;
    c.u_src = u_src;
    c.uH = uH;
    c.uc = (cr && src != SRC_FMG) ? uH : nullptr;
    c.f = f;
    c.u_out = out;
    c.scratch = scratch;
    c.sld = sld;
    launch_smooth_ns2(c, s);
    n_launch++;
  }

  void smooth_into(int l, const T* u_in, const T* f, const T* uc, T* out, cudaStream_t s) {
    const Level& L = lv[l];
    if (d.ns == 1 && !d.nonlinear) {
      VisitDesc<T> v;
      v.src = SRC_LOAD;
      v.cr = uc != nullptr;
      v.epi = false;
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.u_src = u_in;
      v.uc = uc;
      v.f = f;
      v.u_out = out;
      launch_visit(v, s);
    } else {
      ScratchDesc<T> c;
      c.n = L.n;
      c.ld = d.ld;
      c.B = (int)d.B;
      c.W = L.W;
      c.b = L.b;
      c.ns = d.ns;
      c.omega = d.omega;
      c.u_in = u_in;
      c.f = f;
      c.uc = uc;
      c.out = out;
      c.scratch = scratch;
      c.sld = sld;
      c.nonlinear = d.nonlinear != 0;
      launch_smooth_scratch(c, s);
    }
    n_launch++;
  }

  // Top of FMG step t: u_t = Pi u_{t-1}, pre-smooth, restrict + tau to t-1.
  void visit_top(int t, const T* ft, cudaStream_t s) {
    Level& L = lv[t];
    Level& H = lv[t - 1];
    mark_begin(s, t, VK_TOP);
    T* uH_in = H.u[H.cur];
    T* uH_out = H.u[H.cur ^ 1];
    if (fused_restrict_ok(L) || (group_w2(L) && !sharded(t))) {
      VisitDesc<T> v;
      v.src = SRC_FMG;
      v.epi = true;
      v.write_u = !is_sr(t);
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.uH = uH_in;
      v.f = ft;
      v.u_out = L.u[L.cur ^ 1];
      v.uH_out = uH_out;
      v.fH_out = H.f;
      v.E = L.E;
      v.cnt = L.cnt;
      shard_desc(v, t);
      launch_visit(v, s);
      n_launch++;
      if (v.write_u) L.cur ^= 1;
    } else if (fused_chain_ok()) {
      VisitDesc<T> v;  // fused prolongation + smooth, separate restriction
      v.src = SRC_FMG;
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.uH = uH_in;
      v.f = ft;
      v.u_out = L.u[L.cur ^ 1];
      launch_visit(v, s);
      n_launch++;
      L.cur ^= 1;
      launch_restrict_tau(L.u[L.cur], ft, uH_out, H.f, L.n, d.ld, (int)d.B, 2, s, d.nonlinear != 0);
      n_launch++;
    } else if (ns2_ok(L) && L.W >= 4) {  // V(2,2) chain with the restriction fused
      Ns2Desc<T> e;
      e.epi = true;
      e.write_u = !is_sr(t);
      e.uH_out = uH_out;
      e.fH_out = H.f;
      e.E = L.E;
      e.cnt = L.cnt;
      smooth_ns2(t, SRC_FMG, nullptr, uH_in, false, ft, L.u[L.cur ^ 1], s, &e);
      if (e.write_u) L.cur ^= 1;
    } else if (ns2_ok(L)) {
      smooth_ns2(t, SRC_FMG, nullptr, uH_in, false, ft, L.u[L.cur ^ 1], s);
      L.cur ^= 1;
      launch_restrict_tau(L.u[L.cur], ft, uH_out, H.f, L.n, d.ld, (int)d.B, 2, s, d.nonlinear != 0);
      n_launch++;
    } else {
      launch_prolong_fmg(uH_in, tmp, H.n, d.ld, (int)d.B, s);
      n_launch++;
      smooth_into(t, tmp, ft, nullptr, L.u[L.cur ^ 1], s);
      L.cur ^= 1;
      launch_restrict_tau(L.u[L.cur], ft, uH_out, H.f, L.n, d.ld, (int)d.B, 2, s, d.nonlinear != 0);
      n_launch++;
    }
    H.cur ^= 1;
    mark_end(s);
  }

  // Down leg at level l: smooth u_l, restrict + tau to l-1.
  void visit_down(int l, cudaStream_t s) {
    Level& L = lv[l];
    Level& H = lv[l - 1];
    mark_begin(s, l, VK_DOWN);
    // width-2 patches: the group kernel fuses the restriction where the
    // streaming kernel cannot (unsharded / replicated levels only)
    if (fused_restrict_ok(L) || (group_w2(L) && !sharded(l))) {
      VisitDesc<T> v;
      v.src = SRC_LOAD;
      v.epi = true;
      v.write_u = !is_sr(l);
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.u_src = L.u[L.cur];
      v.f = L.f;
      v.u_out = L.u[L.cur ^ 1];
      v.uH_out = (l - 1 == d.m0) ? nullptr : H.u[H.cur ^ 1];
      v.fH_out = H.f;
      v.E = L.E;
      v.cnt = L.cnt;
      shard_desc(v, l);
      launch_visit(v, s);
      n_launch++;
      if (v.write_u) L.cur ^= 1;
      if (v.uH_out) H.cur ^= 1;
    } else if (ns2_ok(L) && L.W >= 4) {
      Ns2Desc<T> e;
      e.epi = true;
      e.write_u = !is_sr(l);
      e.uH_out = (l - 1 == d.m0) ? nullptr : H.u[H.cur ^ 1];
      e.fH_out = H.f;
      e.E = L.E;
      e.cnt = L.cnt;
      smooth_ns2(l, SRC_LOAD, L.u[L.cur], nullptr, false, L.f, L.u[L.cur ^ 1], s, &e);
      if (e.write_u) L.cur ^= 1;
      if (e.uH_out) H.cur ^= 1;
    } else {
      if (ns2_ok(L)) smooth_ns2(l, SRC_LOAD, L.u[L.cur], nullptr, false, L.f, L.u[L.cur ^ 1], s);
      else smooth_into(l, L.u[L.cur], L.f, nullptr, L.u[L.cur ^ 1], s);
      L.cur ^= 1;
      launch_restrict_tau(L.u[L.cur], L.f, H.u[H.cur ^ 1], H.f, L.n, d.ld, (int)d.B, 2, s,
                          d.nonlinear != 0);
      n_launch++;
      H.cur ^= 1;
    }
    mark_end(s);
  }

  // functional output mode (solve_functional): the final up visit reduces
  // J = scale * sum_i w_i u_i instead of writing u_m
  bool fun_mode = false;
  const T* fun_w = nullptr;
  T* fun_out = nullptr;
  T* fun_part = nullptr;  // [P_m][Bp] partial sums
  std::map<std::tuple<const void*, const void*, void*>, cudaGraphExec_t> fgraphs;

  void final_functional(int l, const T* fl, const T* uH, bool sr, cudaStream_t s) {
    Level& L = lv[l];
    const i64 P = L.n / L.W;
    const T scale = fun_w ? T(1) : (T)std::ldexp(1.0, -l);  // unit weights: h * sum u
    if (fused_chain_ok()) {  // the reduction rides in the visit: u_m is never stored
      VisitDesc<T> v;
      v.src = sr ? SRC_FMG : SRC_CORR;
      v.cr = sr;
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.u_src = sr ? nullptr : L.u[L.cur];
      v.uH = uH;
      v.f = fl;
      v.u_out = nullptr;
      v.fun_w = fun_w;
      v.fun_part = fun_part;
      launch_visit(v, s);
    } else {  // other smoothers: the field, then the same ordered reduction
      T* u = L.u[L.cur ^ 1];
      if (ns2_ok(L)) {
        smooth_ns2(l, sr ? SRC_FMG : SRC_CORR, sr ? nullptr : L.u[L.cur], uH, sr, fl, u, s);
      } else {
        Level& H = lv[l - 1];
        if (sr) launch_prolong_fmg(uH, tmp, H.n, d.ld, (int)d.B, s);
        else launch_fas_correct(L.u[L.cur], uH, tmp, L.n, d.ld, (int)d.B, s);
        n_launch++;
        smooth_into(l, tmp, fl, sr ? uH : nullptr, u, s);
      }
      launch_functional_field(u, fun_w, L.n, L.W, d.ld, (int)d.B, fun_part, s);
    }
    n_launch += 2;
    launch_functional_reduce(fun_part, P, (int)d.B, scale, fun_out, s);
  }

  // Up leg at level l: correction (non-SR) or full update + CR (SR), smooth.
  void visit_up(int l, const T* fl, T* dst, cudaStream_t s, bool final = false) {
    Level& L = lv[l];
    Level& H = lv[l - 1];
    mark_begin(s, l, VK_UP);
    T* out = dst ? dst : L.u[L.cur ^ 1];
    const T* uH = H.u[H.cur];
    const bool sr = is_sr(l);
    if (final && fun_mode) {
      final_functional(l, fl, uH, sr, s);
      mark_end(s);
      return;
    }
    if (fused_chain_ok()) {
      VisitDesc<T> v;
      v.src = sr ? SRC_FMG : SRC_CORR;
      v.cr = sr;
      v.n = L.n;
      v.ld = d.ld;
      v.B = (int)d.B;
      v.W = L.W;
      v.b = L.b;
      v.omega = d.omega;
      v.u_src = sr ? nullptr : L.u[L.cur];
      v.uH = uH;
      v.f = fl;
      v.u_out = out;
      shard_desc(v, l);
      launch_visit(v, s);
      n_launch++;
    } else if (ns2_ok(L)) {
      smooth_ns2(l, sr ? SRC_FMG : SRC_CORR, sr ? nullptr : L.u[L.cur], uH, sr, fl, out, s);
    } else {
      if (sr) launch_prolong_fmg(uH, tmp, H.n, d.ld, (int)d.B, s);
      else launch_fas_correct(L.u[L.cur], uH, tmp, L.n, d.ld, (int)d.B, s);
      n_launch++;
      smooth_into(l, tmp, fl, sr ? uH : nullptr, out, s);
    }
    if (!dst) L.cur ^= 1;
    mark_end(s);
  }

  void visit_direct(cudaStream_t s) {
    Level& L = lv[d.m0];
    mark_begin(s, d.m0, VK_DIRECT);
    if (d.nonlinear) launch_direct_solve_nl(L.f, L.u[L.cur ^ 1], L.n, d.ld, (int)d.B, s);
    else launch_direct_solve(L.f, L.u[L.cur ^ 1], L.n, d.ld, (int)d.B, s);
    n_launch++;
    L.cur ^= 1;
    mark_end(s);
  }

  // One full FMG pass (cycles.py:173-214); the level loop of fmg_solve.
  void enqueue(const T* forcing, T* solution, cudaStream_t s) {
    const int m0 = d.m0, m = d.m;
    reset_state(s);
    poison_all(s, forcing_in_place(forcing) ? fm_base : nullptr);
    if (use_coarse) {
      enqueue_coarse(forcing, solution, s);
      return;
    }
    // f cascade (cycles.py:178-180): up to 6 levels per launch
    mark_begin(s, m, VK_CASCADE);
    cascade(forcing, m, m0, false, s);
    mark_end(s);
    n_visit--;  // the cascade is not a level visit
    visit_direct(s);  // cycles.py:183
    for (int k = m0; k < m; k++) {
      const int t = k + 1;
      const T* ft = (t == m) ? forcing : lv[t].f;
      visit_top(t, ft, s);                                 // cycles.py:188-197 (+101-102)
      for (int l = t - 1; l > m0; l--) visit_down(l, s);   // cycles.py:99-105
      visit_direct(s);                                     // smooth_level at m0
      for (int l = m0 + 1; l <= t; l++) {                  // cycles.py:118-133
        const T* fl = (l == m) ? forcing : lv[l].f;
        visit_up(l, fl, (l == m && t == m) ? solution : nullptr, s, l == m && t == m);
      }
      poison_sr_below(t, s);
    }
  }

  void launch_coarse_any(const CoarseArgs<T>& a, cudaStream_t s) {
    if (coarse_warp) launch_coarse_warp(a, d.ns == 2, d.nonlinear != 0, s);
    else launch_coarse(a, s);
  }
  CoarseArgs<T> coarse_args(int mode) const {
    CoarseArgs<T> a;
    a.m0 = d.m0;
    a.Lc = Lc;
    a.m = d.m;
    a.n_sr = d.n_sr;
    a.mode = mode;
    a.CW = CW;
    a.nw = CNW;
    a.pj = (!coarse_warp && Lc > d.m - d.n_sr) ? 1 : 0;
    a.fo = (whole && mode == 0) ? 1 : 0;
    a.B = (int)d.B;
    a.ld = d.ld;
    for (int l = d.m0; l <= Lc; l++) {
      a.W[l] = lv[l].W;
      a.b[l] = lv[l].b;
      a.forig[l] = lv[l].f;
    }
    a.omega = d.omega;
    a.kz.proj_diag = (T)0.5;
    a.kz.recip = (T)2.0;
    a.kz.pow2 = true;
    a.trace = coarse_trace;
    a.f64_arith = mixed ? 1 : 0;
    return a;
  }

  // ---- step schedule (coarse path; the only path that can be sharded) -----------
  // Levels m0..Lc resident in one CTA per column group: one launch for FMG
  // steps m0+1..Lc, then per step t > Lc the grid visits of levels > Lc around
  // one coarse launch for the V-cycle below Lc+1.
  enum StepKind { ST_LOADF, ST_CASCADE_HI, ST_CASCADE_LO, ST_COARSE_FMG, ST_TOP, ST_DOWN,
                  ST_COARSE_V, ST_UP };
  struct Step {
    int kind, l, t;
  };
  std::vector<Step> steps() const {
    std::vector<Step> st;
    if (S > 1) {
      st.push_back({ST_LOADF, d.m, 0});
      st.push_back({ST_CASCADE_HI, d.m, 0});
    }
    if (!whole) st.push_back({ST_CASCADE_LO, d.m, 0});  // whole: the cascade runs on chip
    st.push_back({ST_COARSE_FMG, Lc, 0});  // whole: Lc = m, the loop below is empty
    for (int t = Lc + 1; t <= d.m; t++) {
      st.push_back({ST_TOP, t, t});
      for (int l = t - 1; l > Lc; l--) st.push_back({ST_DOWN, l, t});
      st.push_back({ST_COARSE_V, Lc, t});
      for (int l = Lc + 1; l <= t; l++) st.push_back({ST_UP, l, t});
    }
    return st;
  }
  const T* ffine(const T* forcing) const { return S > 1 ? fm : forcing; }
  const T* flev(int l, const T* forcing) const { return l == d.m ? ffine(forcing) : lv[l].f; }

  void cascade(const T* src, int src_l, int lo_l, bool slab, cudaStream_t s) {
    // restrict levels src_l-1 .. lo_l, up to 6 per launch; slab: this shard's rows
    for (int k = src_l - 1; k >= lo_l;) {
      CascadeDst<T> cd;
      const int sl = k + 1;
      const T* sp = (sl == src_l) ? src : lv[sl].f;
      const i64 r0 = slab ? c0(sl) : 0, nr = slab ? c1(sl) - c0(sl) : lv[sl].n;
      while (cd.levels < 6 && k >= lo_l) {
        cd.p[cd.levels++] = lv[k].f + (slab ? c0(k) : 0) * d.ld;
        k--;
      }
      launch_cascade(sp + r0 * d.ld, nr, cd, d.ld, (int)d.B, s);
      n_launch++;
    }
  }

  void run_step(const Step& st, const T* forcing, T* solution, cudaStream_t s) {
    switch (st.kind) {
      case ST_LOADF:  // the caller's forcing slab into the halo'd finest buffer
        if (!dry && !forcing_in_place(forcing))
          check_cuda(cudaMemcpyAsync(fm + c0(d.m) * d.ld, forcing,
                                   (size_t)(c1(d.m) - c0(d.m)) * d.ld * sizeof(T),
                                   cudaMemcpyDeviceToDevice, s),
                   "forcing slab copy");
        break;
      case ST_CASCADE_HI:  // this shard's slab, finest level down to Lr
        mark_begin(s, d.m, VK_CASCADE);
        cascade(fm, d.m, Lr, true, s);
        mark_end(s);
        n_visit--;
        break;
      case ST_CASCADE_LO: {  // f cascade (cycles.py:178-180) on replicated levels
        const int top = S > 1 ? Lr : d.m;
        mark_begin(s, top, VK_CASCADE);
        cascade(top == d.m ? forcing : lv[top].f, top, d.m0, false, s);
        mark_end(s);
        n_visit--;
        break;
      }
      case ST_COARSE_FMG: {
        mark_begin(s, Lc, VK_COARSE);
        CoarseArgs<T> a = coarse_args(0);
        a.u_top = lv[Lc].u[lv[Lc].cur];
        if (whole) {  // the caller's forcing in, the finest solution out
          a.forig[d.m] = forcing;
          a.u_top = (solution && !fun_mode) ? solution : lv[d.m].u[0];
        }
        launch_coarse_any(a, s);
        n_launch++;
        if (whole && fun_mode) {  // the same ordered reduction as the fused visit
          const Level& L = lv[d.m];
          const T scale = fun_w ? T(1) : (T)std::ldexp(1.0, -d.m);
          launch_functional_field(lv[d.m].u[0], fun_w, L.n, L.W, d.ld, (int)d.B, fun_part, s);
          launch_functional_reduce(fun_part, L.n / L.W, (int)d.B, scale, fun_out, s);
          n_launch += 2;
        }
        mark_end(s);
        break;
      }
      case ST_TOP:
        visit_top(st.l, flev(st.l, forcing), s);
        break;
      case ST_DOWN:
        visit_down(st.l, s);
        break;
      case ST_COARSE_V: {
        mark_begin(s, Lc, VK_COARSE);
        CoarseArgs<T> a = coarse_args(1);
        a.u_top = lv[Lc].u[lv[Lc].cur];  // restricted u_{Lc} in, V-cycled u_{Lc} out (in place)
        a.f_top = lv[Lc].f;
        launch_coarse_any(a, s);
        n_launch++;
        mark_end(s);
        break;
      }
      case ST_UP: {
        const bool fin = st.l == d.m && st.t == d.m;
        T* dst = fin ? (S > 1 ? solution - c0(d.m) * d.ld : solution) : nullptr;
        visit_up(st.l, flev(st.l, forcing), dst, s, fin);
        break;
      }
    }
  }

  // ---- communication after a step (sharded plans) ---------------------------------
  void halo(T* X, int l, int id, std::vector<Xfer>& xs) const {
    const size_t bytes = (size_t)H * d.ld * sizeof(T);
    const i64 a = c0(l), b = c1(l);
    if (srank > 0) {
      xs.push_back({srank - 1, true, X + a * d.ld, bytes, 2 * id, l});
      xs.push_back({srank - 1, false, X + (a - H) * d.ld, bytes, 2 * id + 1, l});
    }
    if (srank < S - 1) {
      xs.push_back({srank + 1, true, X + (b - H) * d.ld, bytes, 2 * id + 1, l});
      xs.push_back({srank + 1, false, X + b * d.ld, bytes, 2 * id, l});
    }
  }
  void records(int l, std::vector<Xfer>& xs) const {
    const i64 slot = 5 * ((d.B + 31) / 32) * 32;
    const size_t bytes = (size_t)slot * sizeof(T);
    if (srank > 0) {
      xs.push_back({srank - 1, true, ob[l], bytes, 0, -1});
      xs.push_back({srank - 1, false, ib[l], bytes, 1, -1});
    }
    if (srank < S - 1) {
      xs.push_back({srank + 1, true, ob[l] + slot, bytes, 1, -1});
      xs.push_back({srank + 1, false, ib[l] + slot, bytes, 0, -1});
    }
  }
  // transfers, slab-edge fix-ups and all-gathers owed after step st
  void comm_plan(const Step& st, std::vector<Xfer>& xs, std::vector<Gather>& gs) const {
    auto gather = [&](T* X, int l) {
      gs.push_back({(char*)X, (size_t)(lv[l].n / S) * d.ld * sizeof(T)});
    };
    switch (st.kind) {
      case ST_LOADF:
        halo(fm, d.m, 1, xs);
        break;
      case ST_CASCADE_HI:
        for (int l = Lr + 1; l < d.m; l++) halo(lv[l].f, l, l, xs);
        gather(lv[Lr].f, Lr);
        break;
      case ST_TOP:
      case ST_DOWN: {
        const int l = st.l;
        if (!sharded(l)) break;
        records(l, xs);
        if (!is_sr(l)) halo(lv[l].u[lv[l].cur], l, 1, xs);
        if (sharded(l - 1)) {
          halo(lv[l - 1].u[lv[l - 1].cur], l - 1, 2, xs);
          halo(lv[l - 1].f, l - 1, 3, xs);
        } else if (l - 1 == Lr) {
          gather(lv[Lr].u[lv[Lr].cur], Lr);
          gather(lv[Lr].f, Lr);
        }
        break;
      }
      case ST_UP:
        if (sharded(st.l) && !(st.l == d.m && st.t == d.m))
          halo(lv[st.l].u[lv[st.l].cur], st.l, 1, xs);
        break;
      default:
        break;
    }
  }
  // the two coarse cells at each slab boundary of an epilogue visit, from the
  // own outbox record and the neighbour's record in the inbox
  void fixup(const Step& st, cudaStream_t s) {
    if (!(st.kind == ST_TOP || st.kind == ST_DOWN) || !sharded(st.l)) return;
    const int l = st.l;
    const i64 slot = 5 * ((d.B + 31) / 32) * 32;
    T* fH = lv[l - 1].f;
    if (c0(l) > 0) {
      launch_edge_fix(ib[l], ob[l], fH, c0(l), lv[l].n, d.ld, (int)d.B, 2, s);
      n_launch++;
    }
    if (c1(l) < lv[l].n) {
      launch_edge_fix(ob[l] + slot, ib[l] + slot, fH, c1(l), lv[l].n, d.ld, (int)d.B, 2, s);
      n_launch++;
    }
  }
  // host-only export of the transport schedule (dry plans): one record per
  // send / recv / all-gather / fix-up, in issue order, after every step
  void schedule(std::vector<fmgsr_comm_rec>& out) {
    reset_state(nullptr);
    int si = 0;
    T* fake = (T*)alloc((size_t)(lv[d.m].n / S) * d.ld * sizeof(T));
    for (const Step& st : steps()) {
      run_step(st, fake, fake, nullptr);
      std::vector<Xfer> xs;
      std::vector<Gather> gs;
      comm_plan(st, xs, gs);
      auto rec = [&](int kind, int peer, int tag, i64 bytes, const void* a, int al) {
        fmgsr_comm_rec r;
        r.step = si;
        r.step_kind = st.kind;
        r.level = st.l;
        r.array_level = al;
        r.pad = 0;
        r.kind = kind;
        r.peer = peer;
        r.tag = tag;
        r.bytes = bytes;
        r.addr = (uint64_t)(uintptr_t)a;
        out.push_back(r);
      };
      for (const Xfer& x : xs)
        rec(x.send ? FMGSR_COMM_SEND : FMGSR_COMM_RECV, x.peer, x.tag, (i64)x.bytes, x.ptr, x.lvl);
      if ((st.kind == ST_TOP || st.kind == ST_DOWN) && sharded(st.l)) {
        const i64 slot = 5 * ((d.B + 31) / 32) * 32;
        if (c0(st.l) > 0) rec(FMGSR_COMM_FIXUP, -1, 0, slot * (i64)sizeof(T), ib[st.l], st.l - 1);
        if (c1(st.l) < lv[st.l].n)
          rec(FMGSR_COMM_FIXUP, -1, 1, slot * (i64)sizeof(T), ib[st.l] + slot, st.l - 1);
      }
      for (const Gather& g : gs) rec(FMGSR_COMM_ALLGATHER, -1, 0, (i64)g.chunk, g.base, Lr);
      si++;
    }
  }
  NcclApi* nccl = nullptr;
  void* ncomm = nullptr;
  void comm_nccl(const Step& st, cudaStream_t s);  // defined after NcclApi

  // ---- peer-memory transport (kernels_p2p.cu) -------------------------------------
  // Every rank maps every peer's plan workspace (CUDA IPC) and pulls: after
  // step si a rank publishes READY, waits for its neighbours' READY, copies
  // their boundary rows / edge records into its own halo rows / inbox (the
  // i-th receive from p reads p's i-th send to this rank, the pairing NCCL
  // uses), runs the slab-edge fix-ups; a gather step then publishes FIXED,
  // waits for every rank's FIXED, copies every rank's chunk of the cutoff
  // level, publishes DONE and waits for every rank's DONE (nobody may touch
  // the replicated level while a peer still reads its chunk).  Sources are
  // resolved once, at import, by replaying each peer's step list on a dry
  // plan of that peer (same allocation sequence, fake addresses) and mapping
  // every address to (allocation index, offset) in the peer's real workspace.
  struct P2pState {
    unsigned long long* flags = nullptr;          // this rank's counter words
    std::vector<unsigned long long*> peer_flags;  // [rank] (own: flags)
    std::vector<void*> opened;                    // IPC mappings
    std::vector<std::vector<const char*>> recv_src;               // [step][receive i]
    std::vector<std::vector<std::vector<const char*>>> gath_src;  // [step][gather][rank]
    unsigned long long timeout_ns = 30ull * 1000000000ull;
    bool ready = false;
  };
  P2pState* p2p = nullptr;
  struct P2pBlob {
    unsigned long long magic, n_alloc, guard, rank;
    cudaIpcMemHandle_t flags;
    cudaIpcMemHandle_t h[1];  // n_alloc handles
  };
  static size_t p2p_blob_bytes(size_t n_alloc) {
    return sizeof(P2pBlob) + (n_alloc ? n_alloc - 1 : 0) * sizeof(cudaIpcMemHandle_t);
  }
  void p2p_init() {
    p2p = new P2pState;
    check_cuda(cudaMalloc(&p2p->flags, P2P_NWORDS * sizeof(unsigned long long)), "p2p flags");
    check_cuda(cudaMemset(p2p->flags, 0, P2P_NWORDS * sizeof(unsigned long long)), "p2p flags");
    if (const char* e = getenv("FMGSR_P2P_TIMEOUT_S")) p2p->timeout_ns = (unsigned long long)(atof(e) * 1e9);
  }
  size_t p2p_export(void* buf, size_t cap) override {
    require(p2p, "p2p_export: not a peer-memory shard plan");
    const size_t need = p2p_blob_bytes(n_init_allocs);
    if (!buf) return need;
    require(cap >= need, "p2p_export: buffer too small");
    std::vector<char> tmpb(need, 0);
    P2pBlob* b = reinterpret_cast<P2pBlob*>(tmpb.data());
    b->magic = 0x46474d5350325031ull;  // "FGMSP2P1"
    b->n_alloc = n_init_allocs;
    b->guard = guards ? GUARD : 0;
    b->rank = (unsigned long long)srank;
    check_cuda(cudaIpcGetMemHandle(&b->flags, p2p->flags), "cudaIpcGetMemHandle (flags)");
    for (size_t k = 0; k < n_init_allocs; k++)
      check_cuda(cudaIpcGetMemHandle(&b->h[k], allocs[k]), "cudaIpcGetMemHandle");
    std::memcpy(buf, tmpb.data(), need);
    return need;
  }
  void p2p_import(const char* all, size_t per_rank) override {
    require(p2p && !p2p->ready, "p2p_import: not a fresh peer-memory shard plan");
    require(per_rank >= p2p_blob_bytes(n_init_allocs), "p2p_import: blob too small");
    // FMGSR_P2P_SELF_PROBE=1 (timing probe on one GPU, results are not a
    // solve): every "peer" is this rank itself -- the S blobs may all be this
    // rank's -- so each wait is met by this rank's own counter and each pull
    // reads this rank's memory at the peer's offsets: the transport's launch,
    // fence, poll and copy cost without a second GPU
    const char* sp = getenv("FMGSR_P2P_SELF_PROBE");
    const bool self_probe = sp && sp[0] == '1';
    // every rank's allocation bases (user pointers) and counter words
    std::vector<std::vector<char*>> base(S);
    p2p->peer_flags.assign(S, nullptr);
    for (int q = 0; q < S; q++) {
      const P2pBlob* b = reinterpret_cast<const P2pBlob*>(all + (size_t)q * per_rank);
      require(b->magic == 0x46474d5350325031ull &&
                  (self_probe || b->rank == (unsigned long long)q),
              "p2p_import: blob of rank " + std::to_string(q) + " is not a shard plan export");
      if (self_probe && q != srank) {
        for (size_t k = 0; k < n_init_allocs; k++) base[q].push_back((char*)alloc_user[k]);
        p2p->peer_flags[q] = p2p->flags;
        continue;
      }
      require(b->n_alloc == n_init_allocs && b->guard == (guards ? GUARD : 0),
              "p2p_import: peer plans differ (descriptor, shard count or FMGSR_GUARDS)");
      if (q == srank) {
        for (size_t k = 0; k < n_init_allocs; k++) base[q].push_back((char*)alloc_user[k]);
        p2p->peer_flags[q] = p2p->flags;
        continue;
      }
      void* fp = nullptr;
      check_cuda(cudaIpcOpenMemHandle(&fp, b->flags, cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle (peer counters)");
      p2p->opened.push_back(fp);
      p2p->peer_flags[q] = (unsigned long long*)fp;
      for (size_t k = 0; k < n_init_allocs; k++) {
        void* ptr = nullptr;
        check_cuda(cudaIpcOpenMemHandle(&ptr, b->h[k], cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle (peer workspace)");
        p2p->opened.push_back(ptr);
        base[q].push_back((char*)ptr + b->guard);
      }
    }
    // replay every rank's step list on a dry plan of that rank
    const std::vector<Step> stl = steps();
    const size_t NS = stl.size();
    std::vector<std::vector<std::vector<Xfer>>> xs_of(S, std::vector<std::vector<Xfer>>(NS));
    std::vector<std::vector<std::vector<Gather>>> gs_of(S, std::vector<std::vector<Gather>>(NS));
    std::vector<std::unique_ptr<Plan<T>>> dryp(S);
    for (int q = 0; q < S; q++) {
      dryp[q].reset(new Plan<T>(d, S, q, true));
      Plan<T>& D = *dryp[q];
      require(D.n_init_allocs == n_init_allocs && D.steps().size() == NS,
              "p2p_import: dry replay differs from the plan");
      D.reset_state(nullptr);
      T* fake = (T*)D.alloc((size_t)(lv[d.m].n / S) * d.ld * sizeof(T));
      size_t si = 0;
      for (const Step& st : D.steps()) {
        D.run_step(st, fake, fake, nullptr);
        D.comm_plan(st, xs_of[q][si], gs_of[q][si]);
        si++;
      }
    }
    auto map = [&](int q, const void* dp) -> const char* {
      const uintptr_t a = (uintptr_t)dp;
      const auto& da = dryp[q]->dry_allocs;
      for (size_t k = 0; k < n_init_allocs; k++)
        if (a >= da[k].first && a < da[k].first + da[k].second)
          return base[q][k] + (a - da[k].first);
      throw Error(ERR_INTERNAL, "p2p_import: transfer address outside the workspace");
    };
    p2p->recv_src.assign(NS, {});
    p2p->gath_src.assign(NS, {});
    for (size_t si = 0; si < NS; si++) {
      std::vector<int> next(S, 0);  // receives from each peer so far in this step
      for (const Xfer& x : xs_of[srank][si]) {
        if (x.send) continue;
        // the i-th send of peer x.peer to this rank
        int i = next[x.peer]++, k = 0;
        const Xfer* src = nullptr;
        for (const Xfer& y : xs_of[x.peer][si])
          if (y.send && y.peer == srank && k++ == i) {
            src = &y;
            break;
          }
        require(src && src->bytes == x.bytes && src->tag == x.tag,
                "p2p_import: unmatched send / receive");
        p2p->recv_src[si].push_back(map(x.peer, src->ptr));
      }
      for (size_t g = 0; g < gs_of[srank][si].size(); g++) {
        std::vector<const char*> per(S);
        for (int q = 0; q < S; q++) {
          require(gs_of[q][si].size() == gs_of[srank][si].size(), "p2p_import: gathers differ");
          per[q] = map(q, gs_of[q][si][g].base);
        }
        p2p->gath_src[si].push_back(per);
      }
    }
    p2p->ready = true;
  }
  int p2p_status() override {
    require(p2p, "p2p_status: not a peer-memory shard plan");
    unsigned long long w[P2P_NWORDS];
    check_cuda(cudaMemcpy(w, p2p->flags, sizeof w, cudaMemcpyDeviceToHost), "p2p status");
    return (int)(w[P2P_ERR] & 0xffffffffu);
  }
  void comm_p2p(const Step& st, int si, cudaStream_t s) {
    if (dry) return;
    require(p2p->ready, "p2p: the peers' workspaces are not imported (fmgsr_shard_p2p_import)");
    std::vector<Xfer> xs;
    std::vector<Gather> gs;
    comm_plan(st, xs, gs);
    if (xs.empty() && gs.empty()) {
      fixup(st, s);
      return;
    }
    const unsigned long long nstep = steps().size() + 1, step = (unsigned long long)si + 1;
    auto copy_base = [&](int which_wait, bool all) {
      P2pCopy c;
      c.nstep = nstep;
      c.step = step;
      c.timeout_ns = p2p->timeout_ns;
      for (int q = 0; q < S; q++) {
        if (q == srank) continue;
        bool need = all;
        for (const Xfer& x : xs) need = need || x.peer == q;
        if (need) c.wait[c.nwait++] = p2p->peer_flags[q] + which_wait;
      }
      return c;
    };
    if (!xs.empty()) {
      P2pCopy c = copy_base(P2P_READY, false);
      c.signal = P2P_READY;
      // this step's slab-edge fix-ups (as fixup()), folded into the kernel
      if ((st.kind == ST_TOP || st.kind == ST_DOWN) && sharded(st.l)) {
        const int l = st.l;
        const i64 Bp = ((d.B + 31) / 32) * 32, slot = 5 * Bp;
        auto add_fix = [&](const T* L, const T* R, i64 sb) {
          P2pFix& x = c.fix[c.nfix++];
          x.L = L;
          x.R = R;
          x.fH = lv[l - 1].f;
          x.s = sb;
          x.nf = lv[l].n;
          x.ld = d.ld;
          x.ldE = Bp;
          x.B = (int)d.B;
        };
        if (c0(l) > 0) add_fix(ib[l], ob[l], c0(l));
        if (c1(l) < lv[l].n) add_fix(ob[l] + slot, ib[l] + slot, c1(l));
      }
      auto overlaps = [](const void* a, size_t na, const void* b, size_t nb) {
        const char *x = (const char*)a, *y = (const char*)b;
        return x < y + nb && y < x + na;
      };
      size_t i = 0;
      for (const Xfer& x : xs) {
        if (x.send) continue;
        require(c.n < P2P_MAXE, "p2p: too many receives in one step");
        c.src[c.n] = p2p->recv_src[si][i++];
        c.dst[c.n] = x.ptr;
        c.bytes[c.n] = x.bytes;
        bool mine = false;  // read or overwritten by a fix-up: CTA 0 copies it first
        for (int k = 0; k < c.nfix; k++) {
          const P2pFix& f = c.fix[k];
          const size_t rec = (size_t)5 * f.ldE * sizeof(T);
          const T* cells = (const T*)f.fH + (f.s / 2 - 1) * f.ld;
          mine = mine || overlaps(x.ptr, x.bytes, f.L, rec) || overlaps(x.ptr, x.bytes, f.R, rec) ||
                 overlaps(x.ptr, x.bytes, cells, (size_t)(f.ld + f.B) * sizeof(T));
        }
        c.cta0[c.n++] = mine;
      }
      launch_p2p_wait_copy<T>(c, p2p->flags, s);
      n_launch++;
    } else {
      fixup(st, s);
    }
    if (!gs.empty()) {
      P2pCopy c = copy_base(P2P_FIXED, true);
      c.signal = P2P_FIXED;
      for (size_t g = 0; g < gs.size(); g++)
        for (int q = 0; q < S; q++) {
          if (q == srank) continue;
          require(c.n < P2P_MAXE, "p2p: too many gather chunks in one step");
          c.src[c.n] = p2p->gath_src[si][g][q] + (size_t)q * gs[g].chunk;
          c.dst[c.n] = gs[g].base + (size_t)q * gs[g].chunk;
          c.bytes[c.n++] = gs[g].chunk;
        }
      for (int e = 0; e < c.n; e++) c.cta0[e] = 0;
      launch_p2p_wait_copy<T>(c, p2p->flags, s);
      P2pCopy dn = copy_base(P2P_DONE, true);
      dn.signal = P2P_DONE;
      launch_p2p_wait_copy<T>(dn, p2p->flags, s);
      n_launch += 2;
    }
  }

  void poison_all(cudaStream_t s, const void* keep = nullptr) {
    if (dry || !(debug & FMGSR_DEBUG_POISON)) return;
    for (size_t k = 0; k < n_field_allocs; k++)
      if (alloc_user[k] != keep) check_cuda(cudaMemsetAsync(alloc_user[k], 0xFF, alloc_sizes[k], s), "poison");
  }
  // after FMG step t: the SR levels below t are dead (levels <= Lc live on chip)
  void poison_sr_below(int t, cudaStream_t s) {
    if (dry || !(debug & FMGSR_DEBUG_POISON)) return;
    for (int l = d.m0; l < t; l++)
      if (is_sr(l) && !(use_coarse && l <= Lc))
        for (int k = 0; k < 2; k++)
          check_cuda(cudaMemsetAsync(lv[l].ub[k], 0xFF, lv[l].ubytes, s), "poison SR level");
  }
  i64 check_guards() override {
    if (!guards) return -1;
    std::vector<unsigned char> h(GUARD);
    i64 bad = 0;
    for (size_t k = 0; k < allocs.size(); k++) {
      const char* lo = (const char*)allocs[k];
      const char* hi = (const char*)alloc_user[k] + alloc_sizes[k];
      for (const char* z : {lo, hi}) {
        check_cuda(cudaMemcpy(h.data(), z, GUARD, cudaMemcpyDeviceToHost), "guard read");
        for (unsigned char c : h) bad += c != 0x5A;
      }
    }
    return bad;
  }
  void set_debug(int flags) override {
    debug = flags;
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);  // recapture with the new flags
    graphs.clear();
    for (auto& kv : fgraphs) cudaGraphExecDestroy(kv.second);
    fgraphs.clear();
  }

  void reset_state(cudaStream_t s) {
    n_launch = 0;
    n_visit = 0;
    for (int l = d.m0; l <= d.m; l++) lv[l].cur = 0;
    if (cnt_bytes) {
      if (!dry) check_cuda(cudaMemsetAsync(cnt_all, 0, cnt_bytes, s), "counter reset");
      n_launch++;
    }
  }

  void enqueue_coarse(const T* forcing, T* solution, cudaStream_t s) {
    if (p2p && !dry) launch_p2p_epoch(p2p->flags, s);
    int si = 0;
    for (const Step& st : steps()) {
      run_step(st, forcing, solution, s);
      if (S > 1) {
        if (p2p) comm_p2p(st, si, s);
        else comm_nccl(st, s);
      }
      if (st.kind == ST_UP && st.l == st.t) poison_sr_below(st.t, s);
      si++;
    }
  }

  void solve(const void* in, void* out, cudaStream_t s) override {
    const T* forcing = (const T*)in;
    T* solution = (T*)out;
    if (!d.use_graph) {
      enqueue(forcing, solution, s);
      return;
    }
    auto key = std::make_pair(in, out);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      cudaGraph_t g;
      check_cuda(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue(forcing, solution, cap);
      } catch (...) {
        cudaStreamEndCapture(cap, &g);
        throw;
      }
      check_cuda(cudaStreamEndCapture(cap, &g), "end capture");
      cudaGraphExec_t ex;
      check_cuda(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
      cudaGraphDestroy(g);
      if (graphs.size() >= 8) {
        cudaGraphExecDestroy(graphs.begin()->second);
        graphs.erase(graphs.begin());
      }
      it = graphs.emplace(key, ex).first;
    }
    check_cuda(cudaGraphLaunch(it->second, s), "graph launch");
  }

  void probe_ms(float* top, float* up) override {
    float* out[2] = {top, up};
    for (int k = 0; k < 2; k++) {
      *out[k] = -1.0f;
      if (!probe_ev[k][0]) continue;
      float ms = 0.0f;
      // events never recorded (finest visit inside the coarse kernel) report not-ready
      if (cudaEventElapsedTime(&ms, probe_ev[k][0], probe_ev[k][1]) == cudaSuccess) *out[k] = ms;
      else cudaGetLastError();
    }
  }

  void solve_functional(const void* in, const void* w, void* out, cudaStream_t s) override {
    require(S == 1, "solve_functional: not available on sharded plans");
    require(!mixed, "solve_functional: not with fp64 arithmetic on fp32 fields");
    if (!fun_part) {  // before any capture: [P_m][Bp] partial sums
      const Level& L = lv[d.m];
      fun_part = alloc((size_t)(L.n / L.W) * (((d.B + 31) / 32) * 32) * sizeof(T));
    }
    auto key = std::make_tuple(in, w, out);
    auto it = fgraphs.find(key);
    fun_w = (const T*)w;
    fun_out = (T*)out;
    fun_mode = true;
    struct Reset {
      bool& m;
      ~Reset() { m = false; }
    } reset{fun_mode};
    if (!d.use_graph) {
      enqueue((const T*)in, nullptr, s);
      return;
    }
    if (it == fgraphs.end()) {
      cudaGraph_t g;
      check_cuda(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue((const T*)in, nullptr, cap);
      } catch (...) {
        cudaStreamEndCapture(cap, &g);
        throw;
      }
      check_cuda(cudaStreamEndCapture(cap, &g), "end capture");
      cudaGraphExec_t ex;
      check_cuda(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
      cudaGraphDestroy(g);
      if (fgraphs.size() >= 8) {
        cudaGraphExecDestroy(fgraphs.begin()->second);
        fgraphs.erase(fgraphs.begin());
      }
      it = fgraphs.emplace(key, ex).first;
    }
    check_cuda(cudaGraphLaunch(it->second, s), "graph launch");
  }

  void solve_timed(const void* in, void* out, cudaStream_t s, float* ms, int32_t* lvl,
                   int32_t* kind, i64 cap_n, i64* nv) override {
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
    ev_lvl.clear();
    ev_kind.clear();
    timing = true;
    try {
      enqueue((const T*)in, (T*)out, s);
    } catch (...) {
      timing = false;
      throw;
    }
    timing = false;
    check_cuda(cudaStreamSynchronize(s), "timed solve sync");
    i64 nvis = (i64)ev_lvl.size();
    *nv = nvis;
    for (i64 i = 0; i < nvis && i < cap_n; i++) {
      float t = 0.f;
      check_cuda(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]), "elapsed");
      ms[i] = t;
      lvl[i] = ev_lvl[i];
      kind[i] = ev_kind[i];
    }
  }

  // Compulsory-traffic model of one solve.
  double words_visit(int kind, int l) const {
    double n = (double)((i64)1 << l);
    switch (kind) {
      case VK_TOP: return 1.0 * n + 0.5 * n + 0.5 * n + 0.5 * n + (is_sr(l) ? 0.0 : n);
      case VK_DOWN: return 2.0 * n + n + (is_sr(l) ? 0.0 : n);
      case VK_UP: return 0.5 * n + n + (is_sr(l) ? 0.0 : n) + n;
      case VK_DIRECT: return 2.0 * n;
      default: return 0.0;
    }
  }
  void info(fmgsr_plan_info* inf) override {
    const int m0 = d.m0, m = d.m;
    double w = (double)((i64)1 << m);  // cascade reads N
    for (int k = m0; k < m; k++) w += (double)((i64)1 << k);  // and writes every coarser f
    i64 visits = 1;
    w += words_visit(VK_DIRECT, m0);
    for (int t = m0 + 1; t <= m; t++) {
      w += words_visit(VK_TOP, t);
      for (int l = t - 1; l > m0; l--) w += words_visit(VK_DOWN, l);
      w += words_visit(VK_DIRECT, m0);
      for (int l = m0 + 1; l <= t; l++) w += words_visit(VK_UP, l);
      visits += 1 + (t - 1 - m0) + 1 + (t - m0);
    }
    inf->workspace_bytes = ws_bytes;
    inf->launches_per_solve = n_launch;
    inf->visits_per_solve = visits;
    inf->alg_bytes_per_solve = w * (double)d.B * sizeof(T);
    inf->finest_visit_alg_bytes = words_visit(VK_UP, m) * (double)d.B * sizeof(T);
    inf->coarse_cutoff = use_coarse ? Lc : -1;
    inf->coarse_columns = use_coarse ? CW : 0;
  }
};

// ---- NCCL, loaded on demand (libnccl.so.2: torch's copy if already loaded) ----------
struct NcclApi {
  typedef int (*GetUniqueId_t)(void*);
  typedef int (*CommInitRank_t)(void**, int, ncclUniqueId, int);
  typedef int (*CommDestroy_t)(void*);
  typedef int (*Group_t)();
  typedef int (*P2P_t)(const void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*Recv_t)(void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*AllGather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
  typedef const char* (*ErrStr_t)(int);
  GetUniqueId_t getUniqueId = nullptr;
  CommInitRank_t commInitRank = nullptr;
  CommDestroy_t commDestroy = nullptr;
  Group_t groupStart = nullptr, groupEnd = nullptr;
  P2P_t send = nullptr;
  Recv_t recv = nullptr;
  AllGather_t allGather = nullptr;
  ErrStr_t errStr = nullptr;
  static NcclApi* get() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
      tried = true;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (h) {
        api.getUniqueId = (GetUniqueId_t)dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (CommInitRank_t)dlsym(h, "ncclCommInitRank");
        api.commDestroy = (CommDestroy_t)dlsym(h, "ncclCommDestroy");
        api.groupStart = (Group_t)dlsym(h, "ncclGroupStart");
        api.groupEnd = (Group_t)dlsym(h, "ncclGroupEnd");
        api.send = (P2P_t)dlsym(h, "ncclSend");
        api.recv = (Recv_t)dlsym(h, "ncclRecv");
        api.allGather = (AllGather_t)dlsym(h, "ncclAllGather");
        api.errStr = (ErrStr_t)dlsym(h, "ncclGetErrorString");
      }
    }
    require(api.commInitRank && api.send && api.allGather, "NCCL (libnccl.so.2) not available");
    return &api;
  }
  void check(int rc, const char* what) const {
    if (rc != 0) throw Error(ERR_CUDA, std::string(what) + ": " + (errStr ? errStr(rc) : "nccl error"));
  }
};

// One shard per GPU: transfers become one grouped ncclSend/ncclRecv round,
// then the slab-edge fix-ups, then in-place ncclAllGather of the cutoff level.
template <typename T>
void Plan<T>::comm_nccl(const Step& st, cudaStream_t s) {
  if (!nccl) {  // local shard plan (timing one shard): no transport, fix-ups still run
    fixup(st, s);
    return;
  }
  std::vector<Xfer> xs;
  std::vector<Gather> gs;
  comm_plan(st, xs, gs);
  if (!xs.empty()) {
    nccl->check(nccl->groupStart(), "ncclGroupStart");
    for (const Xfer& x : xs) {
      if (x.send) nccl->check(nccl->send(x.ptr, x.bytes, ncclUint8, x.peer, ncomm, s), "ncclSend");
      else nccl->check(nccl->recv(x.ptr, x.bytes, ncclUint8, x.peer, ncomm, s), "ncclRecv");
    }
    nccl->check(nccl->groupEnd(), "ncclGroupEnd");
  }
  fixup(st, s);
  for (const Gather& g : gs)
    nccl->check(nccl->allGather(g.base + srank * g.chunk, g.base, g.chunk, ncclUint8, ncomm, s),
                "ncclAllGather");
}

// Virtual shards: S plans of one problem on one device, run in lockstep on one
// stream; the transfers between them are device copies.  Exercises exactly the
// sharded schedule, halos, edge records and cutoff gather of the NCCL path,
// bit-exact against the unsharded solve (tests/test_gpu_shard.py).
struct GroupBase {
  virtual ~GroupBase() {}
  virtual void solve(const void* in, void* out, cudaStream_t s) = 0;
  virtual int cutoff() const = 0;
  virtual i64 halo_rows() const = 0;
};

template <typename T>
struct ShardGroup : GroupBase {
  std::vector<std::unique_ptr<Plan<T>>> sh;
  cudaStream_t cap = nullptr;
  std::map<std::pair<const void*, void*>, cudaGraphExec_t> graphs;
  bool use_graph;
  ShardGroup(const fmgsr_plan_desc& d, int S) : use_graph(d.use_graph != 0) {
    for (int k = 0; k < S; k++) sh.emplace_back(new Plan<T>(d, S, k));
    check_cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "group stream");
  }
  ~ShardGroup() override {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (cap) cudaStreamDestroy(cap);
  }
  int cutoff() const override { return sh[0]->Lr; }
  i64 halo_rows() const override { return sh[0]->H; }
  void enqueue(const T* forcing, T* sol, cudaStream_t s) {
    const int S = (int)sh.size();
    const i64 ld = sh[0]->d.ld;
    for (auto& p : sh) p->reset_state(s);
    for (const auto& st : sh[0]->steps()) {
      std::vector<std::vector<Xfer>> xs(S);
      std::vector<std::vector<Gather>> gs(S);
      for (int k = 0; k < S; k++) {
        const i64 r0 = sh[k]->c0(sh[k]->d.m);
        sh[k]->run_step(st, forcing + r0 * ld, sol + r0 * ld, s);
      }
      for (int k = 0; k < S; k++) sh[k]->comm_plan(st, xs[k], gs[k]);
      // each send lands in the peer's receive exactly as NCCL pairs them: the
      // i-th send k -> p of a group meets the i-th receive at p from k (NCCL
      // p2p has no tags; the tags only assert that the order lines up)
      for (int k = 0; k < S; k++)
        for (int p = 0; p < S; p++) {
          std::vector<const Xfer*> snd, rcv;
          for (const Xfer& x : xs[k])
            if (x.send && x.peer == p) snd.push_back(&x);
          for (const Xfer& y : xs[p])
            if (!y.send && y.peer == k) rcv.push_back(&y);
          require(snd.size() == rcv.size(), "shard group: unmatched transfer count");
          for (size_t i = 0; i < snd.size(); i++) {
            require(snd[i]->tag == rcv[i]->tag && snd[i]->bytes == rcv[i]->bytes,
                    "shard group: send / receive order differs between peers");
            check_cuda(cudaMemcpyAsync(rcv[i]->ptr, snd[i]->ptr, snd[i]->bytes,
                                       cudaMemcpyDeviceToDevice, s), "xfer");
          }
        }
      for (int k = 0; k < S; k++) sh[k]->fixup(st, s);
      for (int k = 0; k < S; k++)
        for (size_t g = 0; g < gs[k].size(); g++)
          for (int j = 0; j < S; j++)
            if (j != k)
              check_cuda(cudaMemcpyAsync(gs[j][g].base + k * gs[k][g].chunk,
                                         gs[k][g].base + k * gs[k][g].chunk, gs[k][g].chunk,
                                         cudaMemcpyDeviceToDevice, s),
                         "gather");
    }
  }
  void solve(const void* in, void* out, cudaStream_t s) override {
    const T* f = (const T*)in;
    T* u = (T*)out;
    if (!use_graph) {
      enqueue(f, u, s);
      return;
    }
    auto key = std::make_pair(in, out);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      cudaGraph_t g;
      check_cuda(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue(f, u, cap);
      } catch (...) {
        cudaStreamEndCapture(cap, &g);
        throw;
      }
      check_cuda(cudaStreamEndCapture(cap, &g), "end capture");
      cudaGraphExec_t ex;
      check_cuda(cudaGraphInstantiate(&ex, g, 0), "graph instantiate");
      cudaGraphDestroy(g);
      it = graphs.emplace(key, ex).first;
    }
    check_cuda(cudaGraphLaunch(it->second, s), "graph launch");
  }
};

static void validate_desc(const fmgsr_plan_desc& d) {
  require(d.m0 >= 2, "m0 must be >= 2 (prolong_fmg needs a coarse field of >= 4 cells)");
  require(d.m > d.m0, "need at least two levels: m must exceed m0");
  require(d.m <= 40, "m too large");
  require(d.n_sr >= 0 && d.n_sr <= d.m - d.m0 - 1, "n_sr outside [0, m - m0 - 1]");
  require(d.ns >= 1, "ns must be >= 1");
  require(d.geom_mode >= 0 && d.geom_mode <= 2, "bad geometry mode");
  require(d.geom_mode != 2 || (d.P >= 1 && is_pow2(d.P)), "P must be a power of two");
  require(d.b >= 0, "buffer must be >= 0");
  require(d.B >= 1 && d.ld >= d.B, "need 1 <= B <= ld");
  require(d.dtype >= 0 && d.dtype <= 2,
          "dtype must be 0 (f64), 1 (f32) or 2 (f32 fields, f64 arithmetic)");
  require(((i64)1 << d.m0) <= 2048, "coarsest level above 2048 cells");
  require(!d.nonlinear || ((i64)1 << d.m0) <= 64, "nonlinear: coarsest level above 64 cells");
}

// ---- fused level visits and the f cascade: helpers of the C entry points --------
static i64 visit_edge_bytes(i64 n, i64 W, i64 B, size_t es) {
  const i64 P = n / W, Bp = (B + 31) / 32 * 32;
  return ((P + 1) * 10 * Bp * (i64)es + 255) / 256 * 256;
}
template <typename T>
static void api_visit_epi(int src, const T* u, const T* uH, const T* f, T* u_out, T* uH_out,
                          T* fH_out, i64 n, i64 B, i64 ld, i64 W, i64 b, double omega,
                          void* work, cudaStream_t s, const char* what) {
  check_field(n, B, ld, what);
  require(W > 0 && n % W == 0, std::string(what) + ": owned width must divide n");
  require(work != nullptr, std::string(what) + ": workspace is null");
  require(fH_out != nullptr, std::string(what) + ": fH_out is null");
  require(!u_out || (u_out != u && u_out != (const T*)f), std::string(what) + ": u_out aliases an input");
  VisitDesc<T> v;
  v.src = src;
  v.cr = false;
  v.epi = true;
  v.write_u = u_out != nullptr;
  v.n = n;
  v.ld = ld;
  v.B = (int)B;
  v.W = W;
  v.b = b;
  v.omega = omega;
  v.u_src = u;
  v.uH = uH;
  v.f = f;
  v.u_out = u_out;
  v.uH_out = uH_out;
  v.fH_out = fH_out;
  v.E = reinterpret_cast<T*>(work);
  v.cnt = reinterpret_cast<int*>(reinterpret_cast<char*>(work) + visit_edge_bytes(n, W, B, sizeof(T)));
  launch_visit(v, s);
}
template <typename T>
static void api_visit_up(const T* u, const T* uH, const T* f, T* u_out, i64 n, i64 B, i64 ld,
                         i64 W, i64 b, int sr, double omega, cudaStream_t s) {
  check_field(n, B, ld, "visit_up");
  require(W > 0 && n % W == 0, "visit_up: owned width must divide n");
  require(u_out != nullptr && u_out != u && u_out != uH, "visit_up: u_out is null or aliases an input");
  VisitDesc<T> v;
  v.src = sr ? SRC_FMG : SRC_CORR;
  v.cr = sr != 0;
  v.n = n;
  v.ld = ld;
  v.B = (int)B;
  v.W = W;
  v.b = b;
  v.omega = omega;
  v.u_src = sr ? nullptr : u;
  v.uH = uH;
  v.f = f;
  v.u_out = u_out;
  launch_visit(v, s);
}
template <typename T>
static void api_f_cascade(const T* f, i64 n, i64 B, i64 ld, int levels, T* const* fo,
                          cudaStream_t s) {
  check_field(n, B, ld, "f_cascade");
  require(f && fo, "f_cascade: null pointer");
  require(levels >= 1 && levels < 63 && (n >> levels) >= 1 && n % ((i64)1 << levels) == 0,
          "f_cascade: levels out of range for n");
  const T* src = f;
  i64 ns = n;
  for (int k = 0; k < levels;) {
    CascadeDst<T> cd;
    while (cd.levels < 6 && k < levels) {
      require(fo[k] != nullptr, "f_cascade: null output level");
      cd.p[cd.levels++] = fo[k++];
    }
    launch_cascade(src, ns, cd, ld, (int)B, s);
    src = cd.p[cd.levels - 1];
    ns >>= cd.levels;
  }
}
}  // namespace fmgsr

using namespace fmgsr;

extern "C" {

int fmgsr_abi_version(void) { return FMGSR_ABI_VERSION; }
const char* fmgsr_last_error(void) { return g_last_error.c_str(); }

#define FMGSR_BOTH(NAME, BODY)                                                         \
  int NAME##_f64 BODY(double) int NAME##_f32 BODY(float)

// ---- kernel lane --------------------------------------------------------------
#define GS_BODY(T)                                                                        \
  (T * u, const T* f, int64_t n, int64_t B, int64_t ld, double inv_h2, int64_t start,      \
   int64_t stop, int forward, double omega, void* stream) {                                \
    return guarded([&] {                                                                  \
      check_field(n, B, ld, "gs_sweep");                                                  \
      launch_gs_sweep<T>(u, f, n, ld, (int)B, inv_h2, start, stop, forward != 0, omega,   \
                         S(stream));                                                      \
    });                                                                                   \
  }
FMGSR_BOTH(fmgsr_gs_sweep, GS_BODY)

#define KZ_BODY(T)                                                                        \
  (T * u, const T* uc, int64_t n, int64_t B, int64_t ld, int64_t start, int64_t stop,      \
   int forward, double proj_diag, void* stream) {                                          \
    (void)forward;                                                                        \
    return guarded([&] {                                                                  \
      check_field(n, B, ld, "kaczmarz_sweep");                                            \
      launch_kaczmarz_sweep<T>(u, uc, n, ld, (int)B, start, stop, proj_diag, S(stream));  \
    });                                                                                   \
  }
FMGSR_BOTH(fmgsr_kaczmarz_sweep, KZ_BODY)

#define SP_BODY(T)                                                                           \
  (const T* u_in, const T* f, T* u_out, int64_t n, int64_t B, int64_t ld, double inv_h2,      \
   const int64_t* olo, const int64_t* ohi, const int64_t* elo, const int64_t* ehi, int64_t P, \
   int64_t ns, double omega, int use_cr, const T* uc, double proj_diag, T* scratch,           \
   const int64_t* soff, int64_t sld, void* stream) {                                          \
    return guarded([&] {                                                                     \
      check_field(n, B, ld, "smooth_patches");                                               \
      require(is_pow2(n) && n >= 2, "smooth_patches: level size must be a power of two");     \
      double want = pow4(level_of(n));                                   \
      require(inv_h2 == want, "smooth_patches: inv_h2 must be 4**level");                     \
      require(u_in != u_out, "smooth_patches: u_out must not alias u_in");                    \
      require(!use_cr || uc != nullptr, "smooth_patches: use_cr needs u_coarse");             \
      if (P == 0) return;                                                                    \
      if (ns == 1) {                                                                         \
        VisitDesc<T> v;                                                                      \
        v.src = SRC_LOAD;                                                                    \
        v.cr = use_cr != 0;                                                                  \
        v.n = n;                                                                             \
        v.ld = ld;                                                                           \
        v.B = (int)B;                                                                        \
        v.omega = omega;                                                                     \
        v.proj_diag = proj_diag;                                                             \
        v.u_src = u_in;                                                                      \
        v.uc = use_cr ? uc : nullptr;                                                        \
        v.f = f;                                                                             \
        v.u_out = u_out;                                                                     \
        v.olo = olo;                                                                         \
        v.ohi = ohi;                                                                         \
        v.elo = elo;                                                                         \
        v.ehi = ehi;                                                                         \
        v.P = P;                                                                             \
        launch_visit(v, S(stream));                                                          \
      } else {                                                                               \
        ScratchDesc<T> c;                                                                    \
        c.n = n;                                                                             \
        c.ld = ld;                                                                           \
        c.B = (int)B;                                                                        \
        c.olo = olo;                                                                         \
        c.ohi = ohi;                                                                         \
        c.elo = elo;                                                                         \
        c.ehi = ehi;                                                                         \
        c.soff = soff;                                                                       \
        c.P = P;                                                                             \
        c.ns = ns;                                                                           \
        c.omega = omega;                                                                     \
        c.proj_diag = proj_diag;                                                             \
        c.u_in = u_in;                                                                       \
        c.f = f;                                                                             \
        c.uc = use_cr ? uc : nullptr;                                                        \
        c.out = u_out;                                                                       \
        c.scratch = scratch;                                                                 \
        c.sld = sld;                                                                         \
        launch_smooth_scratch(c, S(stream));                                                 \
      }                                                                                      \
    });                                                                                      \
  }
FMGSR_BOTH(fmgsr_smooth_patches, SP_BODY)

int64_t fmgsr_smooth_scratch_rows(int64_t n, int64_t W, int64_t b) {
  if (W <= 0 || n <= 0) return 0;
  return scratch_rows_uniform(n, W, b);
}

#define SU_BODY(T)                                                                          \
  (const T* u_in, const T* f, T* u_out, int64_t n, int64_t B, int64_t ld, int64_t W,          \
   int64_t b, int64_t ns, double omega, const T* uc, double proj_diag, T* scratch,            \
   int64_t sld, void* stream) {                                                              \
    return guarded([&] {                                                                    \
      check_field(n, B, ld, "smooth_uniform");                                              \
      require(u_in != u_out, "smooth_uniform: u_out must not alias u_in");                  \
      if (ns == 1 && W % 2 == 0) {                                                          \
        VisitDesc<T> v;                                                                     \
        v.src = SRC_LOAD;                                                                   \
        v.cr = uc != nullptr;                                                               \
        v.n = n;                                                                            \
        v.ld = ld;                                                                          \
        v.B = (int)B;                                                                       \
        v.W = W;                                                                            \
        v.b = b;                                                                            \
        v.omega = omega;                                                                    \
        v.proj_diag = proj_diag;                                                            \
        v.u_src = u_in;                                                                     \
        v.uc = uc;                                                                          \
        v.f = f;                                                                            \
        v.u_out = u_out;                                                                    \
        launch_visit(v, S(stream));                                                         \
      } else {                                                                              \
        ScratchDesc<T> c;                                                                   \
        c.n = n;                                                                            \
        c.ld = ld;                                                                          \
        c.B = (int)B;                                                                       \
        c.W = W;                                                                            \
        c.b = b;                                                                            \
        c.ns = ns;                                                                          \
        c.omega = omega;                                                                    \
        c.proj_diag = proj_diag;                                                            \
        c.u_in = u_in;                                                                      \
        c.f = f;                                                                            \
        c.uc = uc;                                                                          \
        c.out = u_out;                                                                      \
        c.scratch = scratch;                                                                \
        c.sld = sld;                                                                        \
        launch_smooth_scratch(c, S(stream));                                                \
      }                                                                                     \
    });                                                                                     \
  }
FMGSR_BOTH(fmgsr_smooth_uniform, SU_BODY)

// nonlinear smoother (Newton-GS, any ns), staged windows
#define SUNL_BODY(T)                                                                        \
  (const T* u_in, const T* f, T* u_out, int64_t n, int64_t B, int64_t ld, int64_t W,          \
   int64_t b, int64_t ns, double omega, const T* uc, double proj_diag, T* scratch,            \
   int64_t sld, void* stream) {                                                              \
    return guarded([&] {                                                                    \
      check_field(n, B, ld, "smooth_uniform_nl");                                           \
      require(u_in != u_out, "smooth_uniform_nl: u_out must not alias u_in");               \
      ScratchDesc<T> c;                                                                     \
      c.n = n;                                                                              \
      c.ld = ld;                                                                            \
      c.B = (int)B;                                                                         \
      c.W = W;                                                                              \
      c.b = b;                                                                              \
      c.ns = ns;                                                                            \
      c.omega = omega;                                                                      \
      c.proj_diag = proj_diag;                                                              \
      c.u_in = u_in;                                                                        \
      c.f = f;                                                                              \
      c.uc = uc;                                                                            \
      c.out = u_out;                                                                        \
      c.scratch = scratch;                                                                  \
      c.sld = sld;                                                                          \
      c.nonlinear = true;                                                                   \
      launch_smooth_scratch(c, S(stream));                                                  \
    });                                                                                     \
  }
FMGSR_BOTH(fmgsr_smooth_uniform_nl, SUNL_BODY)

// ---- level operators -----------------------------------------------------------
#define OP1(NAME, LAUNCH)                                                                   \
  int NAME##_f64(const double* a, double* out, int64_t n, int64_t B, int64_t ld, void* s) { \
    return guarded([&] { check_field(n, B, ld, #NAME); LAUNCH<double>(a, out, n, ld, (int)B, S(s)); }); \
  }                                                                                         \
  int NAME##_f32(const float* a, float* out, int64_t n, int64_t B, int64_t ld, void* s) {    \
    return guarded([&] { check_field(n, B, ld, #NAME); LAUNCH<float>(a, out, n, ld, (int)B, S(s)); }); \
  }
OP1(fmgsr_apply_operator, launch_apply_operator)
OP1(fmgsr_restrict, launch_restrict)
OP1(fmgsr_prolong_correction, launch_prolong_correction)
OP1(fmgsr_prolong_fmg, launch_prolong_fmg)

int fmgsr_tau_correction_f64(const double* u, double* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "tau"); launch_restrict_tau<double>(u, nullptr, nullptr, out, n, ld, (int)B, 0, S(s)); });
}
int fmgsr_tau_correction_f32(const float* u, float* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "tau"); launch_restrict_tau<float>(u, nullptr, nullptr, out, n, ld, (int)B, 0, S(s)); });
}
int fmgsr_coarse_rhs_f64(const double* f, const double* u, double* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "coarse_rhs"); launch_restrict_tau<double>(u, f, nullptr, out, n, ld, (int)B, 1, S(s)); });
}
int fmgsr_coarse_rhs_f32(const float* f, const float* u, float* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "coarse_rhs"); launch_restrict_tau<float>(u, f, nullptr, out, n, ld, (int)B, 1, S(s)); });
}
int fmgsr_coarse_rhs_nl_f64(const double* f, const double* u, double* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "coarse_rhs_nl"); launch_restrict_tau<double>(u, f, nullptr, out, n, ld, (int)B, 1, S(s), true); });
}
int fmgsr_coarse_rhs_nl_f32(const float* f, const float* u, float* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "coarse_rhs_nl"); launch_restrict_tau<float>(u, f, nullptr, out, n, ld, (int)B, 1, S(s), true); });
}
int fmgsr_direct_solve_nl_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve_nl"); launch_direct_solve_nl<double>(f, u, n, ld, (int)B, S(s)); });
}
int fmgsr_direct_solve_nl_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve_nl"); launch_direct_solve_nl<float>(f, u, n, ld, (int)B, S(s)); });
}
// ---- fused level visits and the f cascade (one call per visit) --------------------
int64_t fmgsr_visit_workspace_bytes(int64_t n, int64_t W, int64_t B, int32_t dtype) {
  if (n <= 0 || W <= 0 || B <= 0 || n % W || (dtype != 0 && dtype != 1)) return 0;
  return visit_edge_bytes(n, W, B, dtype == 0 ? 8 : 4) + (n / W + 1) * ((B + 31) / 32) * 4;
}
#define VISIT_TD(NAME, SRCV, FIRST)                                                            \
  int NAME##_f64(const double* a0, const double* f, double* u_out, double* uH_out,             \
                 double* fH_out, int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b,       \
                 double omega, void* work, void* s) {                                          \
    return guarded([&] {                                                                       \
      api_visit_epi<double>(SRCV, SRCV == SRC_LOAD ? a0 : nullptr, SRCV == SRC_FMG ? a0 : nullptr, \
                            f, u_out, uH_out, fH_out, n, B, ld, W, b, omega, work, S(s), #NAME); \
    });                                                                                        \
  }                                                                                            \
  int NAME##_f32(const float* a0, const float* f, float* u_out, float* uH_out, float* fH_out,  \
                 int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b, double omega,         \
                 void* work, void* s) {                                                        \
    return guarded([&] {                                                                       \
      api_visit_epi<float>(SRCV, SRCV == SRC_LOAD ? a0 : nullptr, SRCV == SRC_FMG ? a0 : nullptr, \
                           f, u_out, uH_out, fH_out, n, B, ld, W, b, omega, work, S(s), #NAME); \
    });                                                                                        \
  }
VISIT_TD(fmgsr_visit_top, SRC_FMG, 0)
VISIT_TD(fmgsr_visit_down, SRC_LOAD, 0)
#undef VISIT_TD
int fmgsr_visit_up_f64(const double* u, const double* uH, const double* f, double* u_out,
                       int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b, int32_t sr,
                       double omega, void* s) {
  return guarded([&] { api_visit_up<double>(u, uH, f, u_out, n, B, ld, W, b, sr, omega, S(s)); });
}
int fmgsr_visit_up_f32(const float* u, const float* uH, const float* f, float* u_out,
                       int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b, int32_t sr,
                       double omega, void* s) {
  return guarded([&] { api_visit_up<float>(u, uH, f, u_out, n, B, ld, W, b, sr, omega, S(s)); });
}
int fmgsr_f_cascade_f64(const double* f, int64_t n, int64_t B, int64_t ld, int32_t levels,
                        double* const* f_out, void* s) {
  return guarded([&] { api_f_cascade<double>(f, n, B, ld, levels, f_out, S(s)); });
}
int fmgsr_f_cascade_f32(const float* f, int64_t n, int64_t B, int64_t ld, int32_t levels,
                        float* const* f_out, void* s) {
  return guarded([&] { api_f_cascade<float>(f, n, B, ld, levels, f_out, S(s)); });
}

int fmgsr_fas_correct_f64(const double* u, const double* uH, double* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "fas_correct"); launch_fas_correct<double>(u, uH, out, n, ld, (int)B, S(s)); });
}
int fmgsr_fas_correct_f32(const float* u, const float* uH, float* out, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "fas_correct"); launch_fas_correct<float>(u, uH, out, n, ld, (int)B, S(s)); });
}
int fmgsr_direct_solve_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve"); launch_direct_solve<double>(f, u, n, ld, (int)B, S(s)); });
}
int fmgsr_direct_solve_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve"); launch_direct_solve<float>(f, u, n, ld, (int)B, S(s)); });
}
int fmgsr_direct_solve_ws_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, double* ws, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve"); require(ws != nullptr, "direct_solve_ws: null workspace"); launch_direct_solve<double>(f, u, n, ld, (int)B, S(s), ws); });
}
int fmgsr_direct_solve_ws_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, float* ws, void* s) {
  return guarded([&] { check_field(n, B, ld, "direct_solve"); require(ws != nullptr, "direct_solve_ws: null workspace"); launch_direct_solve<float>(f, u, n, ld, (int)B, S(s), ws); });
}
int fmgsr_banded_lu_solve_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, double* ws, int* piv, void* s) {
  return guarded([&] { check_field(n, B, ld, "banded_lu_solve"); launch_banded_lu_solve<double>(f, u, n, ld, (int)B, ws, piv, S(s)); });
}
int fmgsr_banded_lu_solve_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, float* ws, int* piv, void* s) {
  return guarded([&] { check_field(n, B, ld, "banded_lu_solve"); launch_banded_lu_solve<float>(f, u, n, ld, (int)B, ws, piv, S(s)); });
}
int fmgsr_nonlinear_rhs_f64(const double* scale, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "nonlinear_rhs"); launch_nonlinear_rhs<double>(scale, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_nonlinear_rhs_f32(const double* scale, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "nonlinear_rhs"); launch_nonlinear_rhs<float>(scale, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_manufactured_rhs_f64(int64_t n, int64_t nmodes, double* f, double* uex, void* s) {
  return guarded([&] { launch_manufactured(n, nmodes, f, uex, S(s)); });
}
int fmgsr_div_check_f64(const double* x, const double* J, double* q, int64_t n, unsigned long long* bad, void* s) {
  return guarded([&] { launch_div_check<double>(x, J, q, n, bad, S(s)); });
}
int fmgsr_div_check_f32(const float* x, const float* J, float* q, int64_t n, unsigned long long* bad, void* s) {
  return guarded([&] { launch_div_check<float>(x, J, q, n, bad, S(s)); });
}
int fmgsr_fourier_rhs_f64(const double* coef, int K, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "fourier_rhs"); launch_fourier_rhs<double>(coef, K, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_fourier_rhs_f32(const double* coef, int K, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "fourier_rhs"); launch_fourier_rhs<float>(coef, K, n, ld, (int)B, f, uex, S(s)); });
}

// ---- plan ------------------------------------------------------------------------
int fmgsr_nccl_unique_id(void* id) {
  return guarded([&] {
    require(id != nullptr, "nccl_unique_id: null argument");
    NcclApi* api = NcclApi::get();
    require(api->getUniqueId != nullptr, "ncclGetUniqueId missing");
    api->check(api->getUniqueId(id), "ncclGetUniqueId");
  });
}
int fmgsr_shard_plan_create(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                            const void* nccl_id, void** plan) {
  return guarded([&] {
    require(desc && plan && nccl_id, "shard_plan_create: null argument");
    validate_desc(*desc);
    require(shards >= 2 && rank >= 0 && rank < shards, "shard_plan_create: bad rank / shards");
    NcclApi* api = NcclApi::get();
    ncclUniqueId uid;
    std::memcpy(&uid, nccl_id, sizeof uid);
    // The plan (every shard-feasibility check -- deterministic, so all ranks
    // agree -- and every allocation) comes first; the collective communicator
    // init only once this rank can run its shard.  RAII frees either on error.
    std::unique_ptr<PlanBase> p;
    if (desc->dtype == 0) p.reset(new Plan<double>(*desc, shards, rank));
    else p.reset(new Plan<float>(*desc, shards, rank));
    void* comm = nullptr;
    api->check(api->commInitRank(&comm, shards, uid, rank), "ncclCommInitRank");
    if (desc->dtype == 0) {
      auto* q = static_cast<Plan<double>*>(p.get());
      q->nccl = api;
      q->ncomm = comm;
    } else {
      auto* q = static_cast<Plan<float>*>(p.get());
      q->nccl = api;
      q->ncomm = comm;
    }
    *plan = p.release();
  });
}
int fmgsr_shard_plan_create_p2p(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                                void** plan) {
  return guarded([&] {
    require(desc && plan, "shard_plan_create_p2p: null argument");
    validate_desc(*desc);
    require(shards >= 2 && rank >= 0 && rank < shards, "shard_plan_create_p2p: bad rank / shards");
    require(shards <= P2P_MAXW + 1, "shard_plan_create_p2p: at most 17 shards");
    std::unique_ptr<PlanBase> p;
    if (desc->dtype == 0) {
      auto* q = new Plan<double>(*desc, shards, rank);
      p.reset(q);
      q->p2p_init();
    } else {
      auto* q = new Plan<float>(*desc, shards, rank);
      p.reset(q);
      q->p2p_init();
    }
    *plan = p.release();
  });
}
int fmgsr_shard_p2p_export(void* plan, void* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    require(plan && len, "shard_p2p_export: null argument");
    auto* p = static_cast<PlanBase*>(plan);
    *len = (int64_t)p->p2p_export(nullptr, 0);
    if (buf) p->p2p_export(buf, (size_t)cap);
  });
}
int fmgsr_shard_p2p_import(void* plan, const void* all, int64_t per_rank) {
  return guarded([&] {
    require(plan && all && per_rank > 0, "shard_p2p_import: null argument");
    static_cast<PlanBase*>(plan)->p2p_import(static_cast<const char*>(all), (size_t)per_rank);
  });
}
int fmgsr_shard_p2p_status(void* plan, int32_t* err) {
  return guarded([&] {
    require(plan && err, "shard_p2p_status: null argument");
    *err = static_cast<PlanBase*>(plan)->p2p_status();
  });
}
int fmgsr_shard_plan_forcing_slab(void* plan, void** slab, int64_t* rows) {
  return guarded([&] {
    require(plan && slab, "shard_plan_forcing_slab: null argument");
    i64 r = 0;
    *slab = static_cast<PlanBase*>(plan)->forcing_slab(&r);
    if (rows) *rows = r;
  });
}
int fmgsr_shard_plan_create_local(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                                  void** plan) {
  return guarded([&] {
    require(desc && plan, "shard_plan_create_local: null argument");
    validate_desc(*desc);
    require(shards >= 2 && rank >= 0 && rank < shards, "shard_plan_create_local: bad rank / shards");
    if (desc->dtype == 0) *plan = new Plan<double>(*desc, shards, rank, false, true);
    else *plan = new Plan<float>(*desc, shards, rank, false, true);
  });
}
int fmgsr_shard_schedule(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                         fmgsr_comm_rec* recs, int64_t cap, int64_t* n, int32_t* cutoff,
                         int64_t* halo_rows) {
  return guarded([&] {
    require(desc && n && cutoff && halo_rows && (recs || cap == 0), "shard_schedule: null argument");
    validate_desc(*desc);
    require(shards >= 2 && rank >= 0 && rank < shards, "shard_schedule: bad rank / shards");
    std::vector<fmgsr_comm_rec> out;
    if (desc->dtype == 0) {
      Plan<double> p(*desc, shards, rank, true);
      p.schedule(out);
      *cutoff = p.Lr;
      *halo_rows = p.H;
    } else {
      Plan<float> p(*desc, shards, rank, true);
      p.schedule(out);
      *cutoff = p.Lr;
      *halo_rows = p.H;
    }
    *n = (int64_t)out.size();
    for (int64_t k = 0; k < cap && k < (int64_t)out.size(); k++) recs[k] = out[k];
  });
}
int fmgsr_shard_group_create(const fmgsr_plan_desc* desc, int32_t shards, void** group) {
  return guarded([&] {
    require(desc && group, "shard_group_create: null argument");
    validate_desc(*desc);
    require(shards >= 2, "shard_group_create: need >= 2 shards");
    if (desc->dtype == 0) *group = new ShardGroup<double>(*desc, shards);
    else *group = new ShardGroup<float>(*desc, shards);
  });
}
int fmgsr_shard_group_solve(void* group, const void* forcing, void* solution, void* stream) {
  return guarded([&] {
    require(group && forcing && solution, "shard_group_solve: null argument");
    reinterpret_cast<GroupBase*>(group)->solve(forcing, solution, S(stream));
  });
}
int fmgsr_shard_group_cutoff(void* group, int32_t* cutoff, int64_t* halo_rows) {
  return guarded([&] {
    require(group && cutoff && halo_rows, "shard_group_cutoff: null argument");
    *cutoff = reinterpret_cast<GroupBase*>(group)->cutoff();
    *halo_rows = reinterpret_cast<GroupBase*>(group)->halo_rows();
  });
}
int fmgsr_shard_group_destroy(void* group) {
  return guarded([&] { delete reinterpret_cast<GroupBase*>(group); });
}
int fmgsr_plan_create(const fmgsr_plan_desc* desc, void** plan) {
  return guarded([&] {
    require(desc && plan, "plan_create: null argument");
    validate_desc(*desc);
    PlanBase* p;
    if (desc->dtype == 0) p = new Plan<double>(*desc);
    else p = new Plan<float>(*desc);
    *plan = p;
  });
}
int fmgsr_plan_set_debug(void* plan, int32_t flags) {
  return guarded([&] {
    require(plan != nullptr, "plan_set_debug: null plan");
    require((flags & ~FMGSR_DEBUG_POISON) == 0, "plan_set_debug: unknown flags");
    reinterpret_cast<PlanBase*>(plan)->set_debug(flags);
  });
}
int fmgsr_plan_check_guards(void* plan, int64_t* bad_bytes) {
  return guarded([&] {
    require(plan && bad_bytes, "plan_check_guards: null argument");
    *bad_bytes = reinterpret_cast<PlanBase*>(plan)->check_guards();
  });
}
int fmgsr_plan_destroy(void* plan) {
  return guarded([&] { delete reinterpret_cast<PlanBase*>(plan); });
}
int fmgsr_plan_get_info(void* plan, fmgsr_plan_info* info) {
  return guarded([&] {
    require(plan && info, "plan_get_info: null argument");
    reinterpret_cast<PlanBase*>(plan)->info(info);
  });
}

int fmgsr_plan_probe_ms(void* plan, float* ms_top, float* ms_up) {
  return guarded([&] {
    require(plan && ms_top && ms_up, "plan_probe_ms: null argument");
    reinterpret_cast<PlanBase*>(plan)->probe_ms(ms_top, ms_up);
  });
}
int fmgsr_plan_solve(void* plan, const void* forcing, void* solution, void* stream) {
  return guarded([&] {
    require(plan && forcing && solution, "plan_solve: null argument");
    require(forcing != solution, "plan_solve: solution must not alias forcing");
    reinterpret_cast<PlanBase*>(plan)->solve(forcing, solution, S(stream));
  });
}
int fmgsr_plan_solve_host(void* plan, const void* h_forcing, void* h_solution, int64_t ld_host,
                          int64_t chunks, void* stream) {
  return fmgsr_plan_solve_host_ex(plan, h_forcing, h_solution, ld_host, chunks, 0, stream);
}
int fmgsr_plan_solve_host_ex(void* plan, const void* h_forcing, void* h_solution, int64_t ld_host,
                             int64_t chunks, int32_t flags, void* stream) {
  return guarded([&] {
    require(plan && h_forcing && h_solution, "plan_solve_host: null argument");
    require((flags & ~FMGSR_HOST_INPUTS_READY) == 0, "plan_solve_host: unknown flags");
    reinterpret_cast<PlanBase*>(plan)->solve_host(h_forcing, h_solution, ld_host, chunks,
                                                  S(stream), flags);
  });
}
int fmgsr_plan_solve_functional(void* plan, const void* forcing, const void* weights,
                                void* functional, void* stream) {
  return guarded([&] {
    require(plan && forcing && functional, "plan_solve_functional: null argument");
    reinterpret_cast<PlanBase*>(plan)->solve_functional(forcing, weights, functional, S(stream));
  });
}
int fmgsr_plan_solve_timed(void* plan, const void* forcing, void* solution, void* stream,
                           float* visit_ms, int32_t* visit_level, int32_t* visit_kind,
                           int64_t cap, int64_t* n_visits) {
  return guarded([&] {
    require(plan && forcing && solution && n_visits, "plan_solve_timed: null argument");
    reinterpret_cast<PlanBase*>(plan)->solve_timed(forcing, solution, S(stream), visit_ms,
                                                   visit_level, visit_kind, cap, n_visits);
  });
}

}  // extern "C"
