// fmgsr_chain.cuh -- the streaming patch chain (ns = 1).
//
// One lane runs the Gauss-Seidel chain of one (patch, rhs): the reference's
// per-patch solve (_kernels_numba.py:79-91) with ns = 1.  Because a single
// forward sweep never lets a cell right of the owned range influence an owned
// cell, the chain stops at the owned end oe (cells [oe, we) are computed and
// discarded by the reference; the cell oe itself is read as frozen data).
// Input pairs come from a PairSource (plain load, FAS correction, or FMG
// prolongation, each with optional just-in-time Kaczmarz), raw loads are
// prefetched PF pairs ahead in registers, and owned results are stored and/or
// pushed into the restriction/tau epilogue.
#pragma once

#include "fmgsr_device.cuh"

namespace fmgsr {

#ifndef FMGSR_PF
#define FMGSR_PF 4
#endif

template <typename T, int SRC, bool CR, bool EPI>
__device__ __forceinline__ void run_chain_ns1(PairSource<T, SRC, CR>& src, const GsCoef<T>& gc,
                                              i64 n, i64 ws, i64 os, i64 oe, T* out, i64 ld,
                                              bool write_u, bool store, Epilogue<T>* epi) {
  constexpr int PF = FMGSR_PF;
  const i64 e = oe;  // cells [ws, e) are updated
  const i64 qs = (ws > 0) ? ((ws - 1) >> 1) : 0;
  const i64 qe = (e - 1) >> 1;

  src.init(qs);
  T v0, v1, f0, f1;
  {
    Raw<T> r = src.load(qs);
    src.make(qs, r, v0, v1);
    f0 = r.f0;
    f1 = r.f1;
  }
  Raw<T> ring[PF];
#pragma unroll
  for (int k = 0; k < PF; k++) ring[k] = src.load(qs + 1 + k);

  T uL = T(0);
  for (i64 q = qs; q <= qe; q += PF) {
#pragma unroll
    for (int k = 0; k < PF; k++) {
      const i64 qq = q + k;
      if (qq <= qe) {
        T w0, w1;
        src.make(qq + 1, ring[k], w0, w1);
        const T g0 = ring[k].f0, g1 = ring[k].f1;
        ring[k] = src.load(qq + 1 + PF);
        const i64 i0 = 2 * qq, i1 = i0 + 1;
        T n0 = v0, n1 = v1;
        if (i0 < ws) {
          uL = v0;  // frozen neighbour of the window
        } else {
          n0 = gs_cell(gc, i0, n, uL, v0, v1, f0);
          uL = n0;
        }
        if (i1 < ws) {
          uL = v1;
        } else if (i1 < e) {
          n1 = gs_cell(gc, i1, n, uL, v1, w0, f1);
          uL = n1;
        }
        if (EPI) {
          if (i0 >= os) {  // owned pairs are whole pairs (os, oe even)
            if (write_u && store) {
              out[i0 * ld] = n0;
              out[i1 * ld] = n1;
            }
            epi->push(qq, n0, n1, f0, f1, store);
          }
        } else if (store) {
          if (i0 >= os && i0 < oe) out[i0 * ld] = n0;
          if (i1 >= os && i1 < oe) out[i1 * ld] = n1;
        }
        v0 = w0;
        v1 = w1;
        f0 = g0;
        f1 = g1;
      }
    }
  }
}

}  // namespace fmgsr
