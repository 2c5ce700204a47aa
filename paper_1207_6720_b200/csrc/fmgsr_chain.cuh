// fmgsr_chain.cuh -- the streaming patch chain (ns = 1).
//
// One lane runs the Gauss-Seidel chain of one (patch, rhs): the reference's
// per-patch solve (_kernels_numba.py:79-91) with ns = 1.  Because a single
// forward sweep never lets a cell right of the owned range influence an owned
// cell, the chain stops at the owned end oe (the reference computes cells
// [oe, we) and discards them; the cell oe itself is read as frozen data).
//
// Input rows are staged D-1 pairs ahead by cp.async into a per-lane ring in
// shared memory (no prefetch registers, one async group per pair).  Pairs
// that touch anything special -- the frozen cell left of the window, domain
// boundary rows, FMG boundary rows, the Kaczmarz window ends, the first two
// owned pairs of the restriction epilogue, clamped loads near the last row --
// go through step_slow(), which evaluates every case like the reference.
// The remaining interior pairs run in fast loops with no per-cell branches
// and pointer-walking addresses.
#pragma once

#include "fmgsr_device.cuh"

#ifndef FMGSR_PROXY_FENCE
#define FMGSR_PROXY_FENCE 0
#endif

namespace fmgsr {

// M: the fields' storage type (T, or fp32 under fp64 arithmetic T)
template <typename T, int SRC, bool CR, bool EPI, bool OMEGA1, int NT, int D, bool BULK,
          bool FUNC = false, typename M = T>
struct Chain {
  static constexpr int R = SrcRows<SRC, CR>::R;
  PairSource<T, SRC, CR, M> src;
  GsCoef<T> gc;
  i64 n, nc, ld, ws, os, oe;
  M* out;  // u_l output, column-offset (nullptr: not written)
  // FUNC: instead of writing the owned cells, accumulate sum_i w_i u_i over
  // them in cell order (w column-offset; nullptr: unit weights)
  const M* fw;
  T facc;
  bool store;
  M* ring;  // this lane's ring: slot s, row k at ring[(s * R + k) * NT]
  Epilogue<T, M>* epi;
  // BULK staging: the warp's D mbarriers; pair x lives in slot x & (D-1) and
  // completes phase ((x - x0) / D) & 1 of that slot's barrier
  unsigned long long* bars;
  int lane;
  i64 x0;
  // chain state: uL = new value left of the current pair; (v0, v1, f0, f1) = current pair
  T uL, v0, v1, f0, f1;

  __device__ __forceinline__ M* slot(i64 x) const { return ring + (i64)((x & (D - 1)) * R) * NT; }

  // stage pair g into slot(g): per-lane cp.async, or one bulk copy per row
  __device__ __forceinline__ void stage(i64 g) {
    if (!BULK) {
      src.template issue<NT>(slot(g), g);
      cp_commit();
      return;
    }
    __syncwarp();  // every lane is done reading this slot's previous pair
    if (lane == 0) {
      const M* p[R];
      src.rows(g, 0, p);
      unsigned long long* bar = bars + (g & (D - 1));
      M* dst = slot(g);  // lane 0: the warp's 32-column segment of each row
      if (FMGSR_PROXY_FENCE) fence_proxy_async();
      mbar_expect_tx(bar, R * 32 * sizeof(M));
#pragma unroll
      for (int k = 0; k < R; k++) bulk_g2s(dst + k * NT, p[k], 32 * sizeof(M), bar);
    }
  }
  // wait until pair g has landed in its slot; AHEAD = g - (the pair whose
  // cells are being updated): pairs up to that pair + D - 1 have been staged
  template <int AHEAD = 1>
  __device__ __forceinline__ void await(i64 g) {
    if (!BULK) {
      cp_wait<D - 1 - AHEAD>();
      return;
    }
    mbar_wait(bars + (g & (D - 1)), (unsigned)(((g - x0) / D) & 1));
  }

  __device__ __forceinline__ T gsi(T l, T u, T r, T f) const {
    T s = xsub(xsub(xmul(T(2), u), l), r);
    T resid = xsub(f, xmul(gc.inv_h2, s));
    if (!OMEGA1) resid = xmul(gc.omega, resid);  // omega == 1: the product is exact
    return xadd(u, xmul(resid, gc.rdiag));
  }

  // general step for pair q (every boundary case, exactly as the reference)
  __device__ __forceinline__ void step_slow(i64 q) {
    await(q + 1);
    Raw<T> r = src.template fetch<NT>(slot(q + 1));
    stage(q + D);
    T w0, w1;
    src.make(q + 1, r, w0, w1);
    const i64 i0 = 2 * q, i1 = i0 + 1;
    T n0 = v0, n1 = v1;
    if (i0 < ws) {
      uL = v0;  // frozen neighbour of the window
    } else {
      n0 = gs_cell(gc, i0, n, uL, v0, v1, f0);
      uL = n0;
    }
    if (i1 < ws) {
      uL = v1;
    } else if (i1 < oe) {
      n1 = gs_cell(gc, i1, n, uL, v1, w0, f1);
      uL = n1;
    }
    if (EPI) {
      if (i0 >= os) {  // owned pairs are whole pairs (os, oe even)
        if (out && store) {
          out[i0 * ld] = cvt<M>(n0);
          out[i1 * ld] = cvt<M>(n1);
        }
        epi->push(q, n0, n1, f0, f1, store);
      }
    } else if (FUNC) {
      if (i0 >= os && i0 < oe) facc = xadd(facc, fw ? xmul(cvt<T>(fw[i0 * ld]), n0) : n0);
      if (i1 >= os && i1 < oe) facc = xadd(facc, fw ? xmul(cvt<T>(fw[i1 * ld]), n1) : n1);
    } else if (store) {
      if (i0 >= os && i0 < oe) out[i0 * ld] = cvt<M>(n0);
      if (i1 >= os && i1 < oe) out[i1 * ld] = cvt<M>(n1);
    }
    v0 = w0;
    v1 = w1;
    f0 = r.f0;
    f1 = r.f1;
  }

  // Fast-loop iteration for pair q with a one-pair lookahead (WIDE shape):
  // wait for pair q+1, stage pair q+D, build pair q+1's smoother input and
  // run the two Gauss-Seidel cells of pair q.
  template <bool KP2>
  __device__ __forceinline__ void it1(i64 q, T& n0, T& n1, T& e0, T& e1) {
    await<1>(q + 1);
    Raw<T> r = src.template fetch<NT>(slot(q + 1));
    if (BULK) {
      stage(q + D);
    } else {
      src.template issue_fast<NT>(slot(q));
      cp_commit();
    }
    T w0, w1;
    src.template make_fast<KP2>(r, w0, w1);
    n0 = gsi(uL, v0, v1, f0);
    n1 = gsi(n0, v1, w0, f1);
    e0 = f0;
    e1 = f1;
    uL = n1;
    v0 = w0;
    v1 = w1;
    f0 = r.f0;
    f1 = r.f1;
  }

  // Fast-loop iteration for pair q with a two-deep lookahead (DEEP shape: a
  // warp issuing alone, where the build of the next pair must not sit between
  // the chain's dependent operations): on entry
  // (v0, v1, f0, f1) is pair q's smoother input and (w0, w1, g0, g1) pair
  // q+1's.  AHEAD: wait for, fetch and build pair q+2 (not on the last pair of
  // the loop, which leaves the source exactly where step_slow expects it).
  // The build of pair q+2 does not depend on the Gauss-Seidel chain of pair
  // q, so the two overlap.  Stages pair q+D into the slot pair q came from.
  // Returns the smoothed cells (n0, n1) and pair q's f (e0, e1).
  template <bool AHEAD, bool KP2>
  __device__ __forceinline__ void it2(i64 q, T& w0, T& w1, T& g0, T& g1, T& n0, T& n1, T& e0,
                                      T& e1) {
    T x0, x1, h0, h1;
    if (AHEAD) {
      await<2>(q + 2);
      Raw<T> r = src.template fetch<NT>(slot(q + 2));
      if (BULK) {
        stage(q + D);
      } else {
        src.template issue_fast<NT>(slot(q));
        cp_commit();
      }
      src.template make_fast<KP2>(r, x0, x1);
      h0 = r.f0;
      h1 = r.f1;
    } else {
      if (BULK) {
        stage(q + D);
      } else {
        src.template issue_fast<NT>(slot(q));
        cp_commit();
      }
    }
    n0 = gsi(uL, v0, v1, f0);
    n1 = gsi(n0, v1, w0, f1);
    e0 = f0;
    e1 = f1;
    uL = n1;
    v0 = w0;
    v1 = w1;
    f0 = g0;
    f1 = g1;
    if (AHEAD) {
      w0 = x0;
      w1 = x1;
      g0 = h0;
      g1 = h1;
    }
  }

  // interior pairs [q, q_end]: OWNED selects store/epilogue, WU the store of
  // the smoothed cells, WUH the epilogue's store of R u.  The epilogue of pair
  // q runs one pair late, inside iteration q+1: its operations depend only on
  // finished values, so they fill the dependency gaps of the next pair's
  // Gauss-Seidel chain instead of waiting on it (the arithmetic of every value
  // is unchanged).  The loop body is one basic block: no per-lane or uniform
  // branches (stores are unconditional, see visit_kernel's rr).
  template <bool OWNED, bool WU, bool WUH, bool KP2>
  __device__ __forceinline__ void run_fast(i64 q, i64 q_end) {
    if (q > q_end) return;
    if (!BULK) src.fast_ptrs(q + D);
    M* po = (OWNED && WU) ? out + (2 * q) * ld : nullptr;
    const M* pw = (FUNC && OWNED && fw) ? fw + (2 * q) * ld : nullptr;
    auto emit = [&](T n0, T n1) {
      if (FUNC && OWNED) {
        if (pw) {
          facc = xadd(facc, xmul(cvt<T>(pw[0]), n0));
          facc = xadd(facc, xmul(cvt<T>(pw[ld]), n1));
          pw += 2 * ld;
        } else {
          facc = xadd(facc, n0);
          facc = xadd(facc, n1);
        }
      } else if (OWNED && WU) {
        po[0] = cvt<M>(n0);
        po[ld] = cvt<M>(n1);
        po += 2 * ld;
      }
    };
    if constexpr (D < 16) {  // one-pair lookahead
      if (EPI && OWNED) {
        epi->fast_begin(q);
        T p0, p1, pf0, pf1;  // the pair whose epilogue is pending
        it1<KP2>(q, p0, p1, pf0, pf1);
        emit(p0, p1);
        for (q++; q <= q_end; q++) {
          T n0, n1, e0, e1;
          epi->template push_fast<WUH>(p0, p1, pf0, pf1);
          it1<KP2>(q, n0, n1, e0, e1);
          emit(n0, n1);
          p0 = n0;
          p1 = n1;
          pf0 = e0;
          pf1 = e1;
        }
        epi->template push_fast<WUH>(p0, p1, pf0, pf1);
        return;
      }
#pragma unroll 2
      for (; q <= q_end; q++) {
        T n0, n1, e0, e1;
        it1<KP2>(q, n0, n1, e0, e1);
        emit(n0, n1);
      }
      return;
    }
    // two-pair lookahead: pair q+1 ahead of the loop
    T w0, w1, g0, g1;
    await<1>(q + 1);
    {
      Raw<T> r = src.template fetch<NT>(slot(q + 1));
      src.template make_fast<KP2>(r, w0, w1);
      g0 = r.f0;
      g1 = r.f1;
    }
    if (EPI && OWNED) {
      epi->fast_begin(q);
      T p0, p1, pf0, pf1;  // the pair whose epilogue is pending
      if (q == q_end) {
        it2<false, KP2>(q, w0, w1, g0, g1, p0, p1, pf0, pf1);
      } else {
        it2<true, KP2>(q, w0, w1, g0, g1, p0, p1, pf0, pf1);
        emit(p0, p1);
#pragma unroll 2
        for (q++; q < q_end; q++) {
          T n0, n1, e0, e1;
          epi->template push_fast<WUH>(p0, p1, pf0, pf1);
          it2<true, KP2>(q, w0, w1, g0, g1, n0, n1, e0, e1);
          emit(n0, n1);
          p0 = n0;
          p1 = n1;
          pf0 = e0;
          pf1 = e1;
        }
        T n0, n1, e0, e1;
        epi->template push_fast<WUH>(p0, p1, pf0, pf1);
        it2<false, KP2>(q, w0, w1, g0, g1, n0, n1, e0, e1);
        p0 = n0;
        p1 = n1;
        pf0 = e0;
        pf1 = e1;
      }
      emit(p0, p1);
      epi->template push_fast<WUH>(p0, p1, pf0, pf1);
      return;
    }
#pragma unroll 2
    for (; q < q_end; q++) {
      T n0, n1, e0, e1;
      it2<true, KP2>(q, w0, w1, g0, g1, n0, n1, e0, e1);
      emit(n0, n1);
    }
    T n0, n1, e0, e1;
    it2<false, KP2>(q, w0, w1, g0, g1, n0, n1, e0, e1);
    emit(n0, n1);
  }
  template <bool OWNED, bool KP2>
  __device__ __forceinline__ void run_fast_k(i64 q, i64 q_end) {
    if (!OWNED) {
      run_fast<false, false, false, KP2>(q, q_end);
    } else if (EPI) {
      const bool wu = out != nullptr, wuh = epi->write_uH;
      if (wu && wuh) run_fast<true, true, true, KP2>(q, q_end);
      else if (wu) run_fast<true, true, false, KP2>(q, q_end);
      else if (wuh) run_fast<true, false, true, KP2>(q, q_end);
      else run_fast<true, false, false, KP2>(q, q_end);
    } else {
      if (out) run_fast<true, true, false, KP2>(q, q_end);
      else run_fast<true, false, false, KP2>(q, q_end);
    }
  }
  template <bool OWNED>
  __device__ __forceinline__ void run_fast_any(i64 q, i64 q_end) {
    if (!CR || src.kz.pow2) run_fast_k<OWNED, true>(q, q_end);
    else run_fast_k<OWNED, false>(q, q_end);
  }

  __device__ __forceinline__ void run(i64 we) {
    const i64 qs = (ws > 0) ? ((ws - 1) >> 1) : 0;
    const i64 qe = (oe - 1) >> 1;
    // chain head: the direct loads of the state before pair qs and of pair qs
    // gate the chain, so they are issued first; the D-1 staged pairs follow
    // while they are in flight (one memory latency for the whole head)
    x0 = qs + 1;
    src.init_loads(qs);
    Raw<T> r0 = src.load(qs);
    for (int k = 1; k < D; k++) stage(qs + k);
    src.init_finish(qs);
    src.make(qs, r0, v0, v1);
    f0 = r0.f0;
    f1 = r0.f1;
    uL = T(0);
    // interior range: both cells updated and interior, generation of q+1
    // interior, CR window interior, unclamped fast issue of q + D
    i64 lo = (ws + 1) >> 1;
    if (lo < 1) lo = 1;
    i64 hi = (oe - 2) >> 1;
    if (hi > nc - 2) hi = nc - 2;
    if (SRC == SRC_FMG) hi = hi < nc - 4 ? hi : nc - 4;
    if (SRC == SRC_CORR) hi = hi < nc - 3 ? hi : nc - 3;
    if (CR) {
      const i64 a = src.wlo - 1, b = (we >> 1) - 2;
      lo = lo > a ? lo : a;
      hi = hi < b ? hi : b;
    }
    hi = hi < src.qhi - 2 - D ? hi : src.qhi - 2 - D;  // unclamped fast issue stays in memory
    const i64 oq = os >> 1;
    i64 q = qs;
    // buffer cells left of the owned range
    const i64 bl = lo, bh = hi < oq - 1 ? hi : oq - 1;
    if (bl <= bh) {
      for (; q < bl; q++) step_slow(q);
      run_fast_any<false>(q, bh);
      q = bh + 1;
    }
    // owned cells
    const i64 ol = lo > oq + (EPI ? 2 : 0) ? lo : oq + (EPI ? 2 : 0);
    if (ol <= hi) {
      for (; q < ol; q++) step_slow(q);
      run_fast_any<true>(q, hi);
      q = hi + 1;
    }
    for (; q <= qe; q++) step_slow(q);
    if (BULK) {
      // drain the pairs still in flight before the CTA may exit
      for (i64 g = qe + 2; g <= qe + D; g++) await(g);
    } else {
      cp_wait<0>();
    }
  }
};

}  // namespace fmgsr
