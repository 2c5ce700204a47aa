// capi.cu -- extern "C" boundary of libfmgsr_cuda.so (include/fmgsr_cuda.h)
// and the native FMG-FAS(-SR) solve plan.
//
// The plan is the B200-side replacement of the reference driver
// (cycles.py:95-222): it owns the per-level device workspace, derives the
// level-visit schedule once, emits one fused kernel per level visit where
// the visit qualifies (ns = 1, owned width >= 4 for visits that restrict),
// and captures the whole cycle into a CUDA graph that is replayed per solve.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fmgsr_cuda.h"
#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

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

struct PlanBase {
  fmgsr_plan_desc d{};
  virtual ~PlanBase() {}
  virtual void solve(const void* in, void* out, cudaStream_t s) = 0;
  virtual void solve_timed(const void* in, void* out, cudaStream_t s, float* ms, int32_t* lvl,
                           int32_t* kind, i64 cap, i64* nv) = 0;
  virtual void info(fmgsr_plan_info* inf) = 0;
  virtual void solve_host(const void* h_in, void* h_out, i64 ld_host, i64 chunks,
                          cudaStream_t s) = 0;
};

template <typename T>
struct Plan : PlanBase {
  struct Level {
    i64 n = 0, W = 0, b = 0;
    T* u[2] = {nullptr, nullptr};
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
  std::vector<void*> allocs;
  i64 ws_bytes = 0;
  cudaStream_t cap = nullptr;
  std::map<std::pair<const void*, void*>, cudaGraphExec_t> graphs;
  // per-solve bookkeeping (filled by enqueue)
  i64 n_launch = 0, n_visit = 0;
  // timing hooks
  std::vector<cudaEvent_t> ev;
  std::vector<int32_t> ev_lvl, ev_kind;
  bool timing = false;
  // coarse hierarchy kernel: levels m0..Lc on chip, CW RHS columns per CTA
  bool use_coarse = false;
  int Lc = 0, CW = 1;
  int coarse_trace = 0;

  bool is_sr(int l) const { return l > d.m - d.n_sr; }

  T* alloc(size_t bytes) {
    void* p = nullptr;
    check_cuda(cudaMalloc(&p, bytes ? bytes : 16), "plan workspace cudaMalloc");
    allocs.push_back(p);
    ws_bytes += (i64)bytes;
    return (T*)p;
  }

  explicit Plan(const fmgsr_plan_desc& desc) {
    d = desc;
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
      if (l > m0 && L.W >= 4) cnt_total += (L.n / L.W + 1) * nrg;
    }
    for (int l = m0; l <= m; l++) {
      Level& L = lv[l];
      size_t fb = (size_t)L.n * ld * sizeof(T);
      L.u[0] = alloc(fb);
      L.u[1] = alloc(fb);
      if (l < m) L.f = alloc(fb);
      if (l > m0 && L.W >= 4) L.E = alloc((size_t)(L.n / L.W + 1) * 10 * Bp * sizeof(T));
    }
    tmp = alloc((size_t)tmp_rows * ld * sizeof(T));
    if (scratch_rows) {
      sld = Bp;
      scratch = alloc((size_t)scratch_rows * sld * sizeof(T));
    }
    cnt_bytes = (size_t)cnt_total * sizeof(int);
    cnt_all = (int*)alloc(cnt_bytes);
    check_cuda(cudaMemset(cnt_all, 0, cnt_bytes ? cnt_bytes : 16), "plan memset");
    i64 off = 0;
    for (int l = m0 + 1; l <= m; l++) {
      Level& L = lv[l];
      if (L.W >= 4) {
        L.cnt = cnt_all + off;
        off += (L.n / L.W + 1) * nrg;
      }
    }
    check_cuda(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "plan stream");
    // Coarse cutoff: about 128 CTAs of CW columns; the deepest level whose
    // three fields per level (two u, f) for CW columns fit in ~200 KB.
    use_coarse = d.fused && d.ns == 1 && d.coarse != 0 && !d.nonlinear;
    const char* tr = getenv("FMGSR_COARSE_TRACE");
    coarse_trace = (tr && tr[0] == '1') ? 1 : 0;
    if (use_coarse) {
      i64 cw = 1;
      // ~128 CTAs (one wave on 148 SMs); measured best against 256 / 512
      i64 target = 128;
      if (const char* e = getenv("FMGSR_COARSE_CTAS")) target = atoll(e);
      while (cw * 2 <= 32 && cw * 2 * target <= d.B) cw *= 2;
      CW = (int)cw;
      Lc = m0;
      while (Lc + 1 <= m - 1 && coarse_smem_bytes<T>(m0, Lc + 1, CW) <= 200 * 1024) Lc++;
      int want = d.coarse;
      if (want < 0)
        if (const char* e = getenv("FMGSR_COARSE_LC")) want = atoi(e) + 1;
      if (want > 0 && want - 1 >= m0 && want - 1 < Lc) Lc = want - 1;
    }
  }

  ~Plan() override {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : hev) cudaEventDestroy(e);
    if (cap) cudaStreamDestroy(cap);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    for (void* p : allocs) cudaFree(p);
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

  void solve_host(const void* h_in, void* h_out, i64 ld_host, i64 chunks,
                  cudaStream_t s) override {
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
    // the caller's stream orders us after its prior work
    for (int k = 0; k < 2; k++) {
      check_cuda(cudaEventRecord(solved[k], s), "ev");
      check_cuda(cudaEventRecord(out_done[k], s), "ev");
    }
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
  void mark_begin(cudaStream_t s, int lvl, int kind) {
    n_visit++;
    if (!timing) return;
    cudaEvent_t a;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventRecord(a, s), "event record");
    ev.push_back(a);
    ev_lvl.push_back(lvl);
    ev_kind.push_back(kind);
  }
  void mark_end(cudaStream_t s) {
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
    if (fused_restrict_ok(L)) {
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
    if (fused_restrict_ok(L)) {
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
      launch_visit(v, s);
      n_launch++;
      if (v.write_u) L.cur ^= 1;
      if (v.uH_out) H.cur ^= 1;
    } else {
      smooth_into(l, L.u[L.cur], L.f, nullptr, L.u[L.cur ^ 1], s);
      L.cur ^= 1;
      launch_restrict_tau(L.u[L.cur], L.f, H.u[H.cur ^ 1], H.f, L.n, d.ld, (int)d.B, 2, s,
                          d.nonlinear != 0);
      n_launch++;
      H.cur ^= 1;
    }
    mark_end(s);
  }

  // Up leg at level l: correction (non-SR) or full update + CR (SR), smooth.
  void visit_up(int l, const T* fl, T* dst, cudaStream_t s) {
    Level& L = lv[l];
    Level& H = lv[l - 1];
    mark_begin(s, l, VK_UP);
    T* out = dst ? dst : L.u[L.cur ^ 1];
    const T* uH = H.u[H.cur];
    const bool sr = is_sr(l);
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
      launch_visit(v, s);
      n_launch++;
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
    n_launch = 0;
    n_visit = 0;
    for (int l = m0; l <= m; l++) lv[l].cur = 0;
    if (cnt_bytes) {
      check_cuda(cudaMemsetAsync(cnt_all, 0, cnt_bytes, s), "counter reset");
      n_launch++;
    }
    // f cascade (cycles.py:178-180): up to 6 levels per launch
    mark_begin(s, m, VK_CASCADE);
    for (int k = m - 1; k >= m0;) {
      CascadeDst<T> cd;
      const int src_l = k + 1;
      const T* src = (src_l == m) ? forcing : lv[src_l].f;
      while (cd.levels < 6 && k >= m0) cd.p[cd.levels++] = lv[k--].f;
      launch_cascade(src, (i64)1 << src_l, cd, d.ld, (int)d.B, s);
      n_launch++;
    }
    mark_end(s);
    n_visit--;  // the cascade is not a level visit
    if (use_coarse) {
      enqueue_coarse(forcing, solution, s);
      return;
    }
    visit_direct(s);  // cycles.py:183
    for (int k = m0; k < m; k++) {
      const int t = k + 1;
      const T* ft = (t == m) ? forcing : lv[t].f;
      visit_top(t, ft, s);                                 // cycles.py:188-197 (+101-102)
      for (int l = t - 1; l > m0; l--) visit_down(l, s);   // cycles.py:99-105
      visit_direct(s);                                     // smooth_level at m0
      for (int l = m0 + 1; l <= t; l++) {                  // cycles.py:118-133
        const T* fl = (l == m) ? forcing : lv[l].f;
        visit_up(l, fl, (l == m && t == m) ? solution : nullptr, s);
      }
    }
  }

  CoarseArgs<T> coarse_args(int mode) const {
    CoarseArgs<T> a;
    a.m0 = d.m0;
    a.Lc = Lc;
    a.m = d.m;
    a.n_sr = d.n_sr;
    a.mode = mode;
    a.CW = CW;
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
    return a;
  }

  // Schedule with levels m0..Lc resident in one CTA per column group: one
  // launch for FMG steps m0+1..Lc, then per step t > Lc the grid visits of
  // levels > Lc around one coarse launch for the V-cycle below Lc+1.
  void enqueue_coarse(const T* forcing, T* solution, cudaStream_t s) {
    const int m = d.m;
    {
      mark_begin(s, Lc, VK_COARSE);
      CoarseArgs<T> a = coarse_args(0);
      a.u_top = lv[Lc].u[lv[Lc].cur];
      launch_coarse(a, s);
      n_launch++;
      mark_end(s);
    }
    for (int t = Lc + 1; t <= m; t++) {
      const T* ft = (t == m) ? forcing : lv[t].f;
      visit_top(t, ft, s);
      for (int l = t - 1; l > Lc; l--) visit_down(l, s);
      mark_begin(s, Lc, VK_COARSE);
      CoarseArgs<T> a = coarse_args(1);
      a.u_top = lv[Lc].u[lv[Lc].cur];  // restricted u_{Lc} in, V-cycled u_{Lc} out (in place)
      a.f_top = lv[Lc].f;
      launch_coarse(a, s);
      n_launch++;
      mark_end(s);
      for (int l = Lc + 1; l <= t; l++) {
        const T* fl = (l == m) ? forcing : lv[l].f;
        visit_up(l, fl, (l == m && t == m) ? solution : nullptr, s);
      }
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
  require(d.dtype == 0 || d.dtype == 1, "dtype must be 0 (f64) or 1 (f32)");
  require(((i64)1 << d.m0) <= 2048, "coarsest level above 2048 cells");
  require(!d.nonlinear || ((i64)1 << d.m0) <= 64, "nonlinear: coarsest level above 64 cells");
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
      double want = (double)((i64)1 << (2 * level_of(n)));                                   \
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
int fmgsr_nonlinear_rhs_f64(const double* scale, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "nonlinear_rhs"); launch_nonlinear_rhs<double>(scale, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_nonlinear_rhs_f32(const double* scale, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "nonlinear_rhs"); launch_nonlinear_rhs<float>(scale, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_fourier_rhs_f64(const double* coef, int K, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "fourier_rhs"); launch_fourier_rhs<double>(coef, K, n, ld, (int)B, f, uex, S(s)); });
}
int fmgsr_fourier_rhs_f32(const double* coef, int K, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* s) {
  return guarded([&] { check_field(n, B, ld, "fourier_rhs"); launch_fourier_rhs<float>(coef, K, n, ld, (int)B, f, uex, S(s)); });
}

// ---- plan ------------------------------------------------------------------------
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
int fmgsr_plan_destroy(void* plan) {
  return guarded([&] { delete reinterpret_cast<PlanBase*>(plan); });
}
int fmgsr_plan_get_info(void* plan, fmgsr_plan_info* info) {
  return guarded([&] {
    require(plan && info, "plan_get_info: null argument");
    reinterpret_cast<PlanBase*>(plan)->info(info);
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
  return guarded([&] {
    require(plan && h_forcing && h_solution, "plan_solve_host: null argument");
    reinterpret_cast<PlanBase*>(plan)->solve_host(h_forcing, h_solution, ld_host, chunks,
                                                  S(stream));
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
