// kernels_p2p.cu -- peer-memory transport of the patch-slab sharded plan.
//
// The NCCL transport (capi.cu comm_nccl) turns each exchange of the sharded
// schedule into a grouped ncclSend / ncclRecv round.  This transport needs no
// collective library: every rank maps its peers' plan workspaces (CUDA IPC
// handles, NVLink peer access between GPUs) and PULLS what it needs -- the
// neighbours' boundary rows and tau edge records, every rank's chunk of the
// replication-cutoff level -- straight into its own halo / inbox / replicated
// arrays.  All writes are local; only reads cross the link, so no rank ever
// writes into memory a peer is still reading.  Ordering is three monotonic
// per-rank counters in device memory (READY after a rank's visit, FIXED after
// its slab-edge fix-ups, DONE after its gather), published with
// st.release.sys and polled with ld.acquire.sys; a step's value is
// epoch * steps_per_solve + step, and the epoch advances once per solve on
// the device (so captured CUDA graphs replay unchanged).
#include <cstdint>

#include "fmgsr_device.cuh"
#include "fmgsr_internal.h"

namespace fmgsr {

namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_p2p_epoch(unsigned long long* flags) {
  if (blockIdx.x == 0 && threadIdx.x == 0) flags[P2P_EPOCH] += 1;
}

// CTA 0 first publishes this rank's counter c.signal (if >= 0); thread 0 of
// every CTA then polls the listed peer counters until they reach this step's
// value (bounded: past the timeout the error word is set and nothing is
// copied, so a broken peer cannot hang the GPU); then the CTAs copy every
// (remote source, local destination) pair, 16 bytes per thread and load,
// through L2 only (ld.global.cg: a peer's rows are never served stale from
// L1).  The slab-edge fix-ups of the step (c.fix) run in CTA 0 after it has
// copied, by itself, every entry they read or overwrite (the edge records,
// the halo rows of f_H holding the neighbour's boundary cell) -- one launch
// per exchange round instead of three.
template <typename T>
__global__ void k_p2p_wait_copy(P2pCopy c, unsigned long long* flags) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const unsigned long long v = flags[P2P_EPOCH] * c.nstep + c.step;
    // publish this rank's counter first (this launch follows the step's
    // kernels in stream order, so their writes are complete), then wait
    if (c.signal >= 0 && blockIdx.x == 0) {
      __threadfence_system();
      st_release_sys(flags + c.signal, v);
    }
    int good = 1;
    for (int k = 0; k < c.nwait && good; k++) {
      const unsigned long long t0 = globaltimer_ns();
      while (ld_acquire_sys(c.wait[k]) < v) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > c.timeout_ns) {
          good = 0;
          atomicExch(reinterpret_cast<unsigned int*>(flags + P2P_ERR), 1u);
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();  // orders every thread's loads below after thread 0's acquire
  if (!ok) return;
  auto copy = [](const void* src, void* dst, unsigned long long bytes, unsigned long long tid,
                 unsigned long long nth) {
    // four independent 16-byte loads in flight per thread before their stores:
    // the copy is latency-bound (a link round trip per pass)
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    const unsigned long long w = bytes >> 4;
    for (unsigned long long i = tid; i < w; i += 4 * nth) {
      uint4 v[4];
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (i + k * nth < w) v[k] = __ldcg(s + i + k * nth);
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (i + k * nth < w) d[i + k * nth] = v[k];
    }
  };
  const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long gth = (unsigned long long)gridDim.x * blockDim.x;
  for (int e = 0; e < c.n; e++) {
    if (c.cta0[e]) {
      if (blockIdx.x == 0) copy(c.src[e], c.dst[e], c.bytes[e], threadIdx.x, blockDim.x);
    } else {
      copy(c.src[e], c.dst[e], c.bytes[e], gtid, gth);
    }
  }
  if (blockIdx.x != 0 || c.nfix == 0) return;
  __syncthreads();
  for (int k = 0; k < c.nfix; k++) {
    const P2pFix& x = c.fix[k];
    const T* L = static_cast<const T*>(x.L);
    const T* R = static_cast<const T*>(x.R);
    T* fH = static_cast<T*>(x.fH);
    const int lv = level_of(x.nf);
    const T ih = (T)pow4(lv), iH = (T)pow4(lv - 1);
    for (int r = threadIdx.x; r < x.B; r += blockDim.x) {
      T Lr[5], Rr[5];
#pragma unroll
      for (int q = 0; q < 5; q++) {
        Lr[q] = L[q * x.ldE + r];
        Rr[q] = R[q * x.ldE + r];
      }
      T fL, fR;
      edge_finish(Lr, Rr, ih, iH, fL, fR);
      fH[(x.s / 2 - 1) * x.ld + r] = fL;
      fH[(x.s / 2) * x.ld + r] = fR;
    }
  }
}

}  // namespace

void launch_p2p_epoch(unsigned long long* flags, cudaStream_t s) {
  k_p2p_epoch<<<1, 32, 0, s>>>(flags);
  check_launch("p2p_epoch");
}
template <typename T>
void launch_p2p_wait_copy(const P2pCopy& c, unsigned long long* flags, cudaStream_t s) {
  require(c.n >= 0 && c.n <= P2P_MAXE && c.nwait >= 0 && c.nwait <= P2P_MAXW &&
              c.nfix >= 0 && c.nfix <= 2,
          "p2p: too many transfers in one step");
  unsigned long long total = 0;
  for (int e = 0; e < c.n; e++) {
    require(c.bytes[e] % 16 == 0 && ((uintptr_t)c.src[e] & 15) == 0 &&
                ((uintptr_t)c.dst[e] & 15) == 0,
            "p2p: transfers must be 16-byte aligned multiples of 16 bytes");
    if (!c.cta0[e]) total += c.bytes[e];
  }
  // ~16 KB per CTA (one pass of four loads per thread), at most one CTA per SM
  // (every CTA polls the counters)
  unsigned long long blocks = (total + 16383) / 16384;
  if (blocks < 1) blocks = 1;
  if (blocks > 148) blocks = 148;
  k_p2p_wait_copy<T><<<(unsigned)blocks, 256, 0, s>>>(c, flags);
  check_launch("p2p_wait_copy");
}
template void launch_p2p_wait_copy<double>(const P2pCopy&, unsigned long long*, cudaStream_t);
template void launch_p2p_wait_copy<float>(const P2pCopy&, unsigned long long*, cudaStream_t);

}  // namespace fmgsr
