// PCIe bandwidth on the box: 1D / 2D (column-chunk rows) H2D, D2H, and both at once.
#include <cstdio>
#include <cuda_runtime.h>
// SM-driven copy over PCIe (pinned host memory is device-addressable under UVA)
__global__ void kcopy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
int main() {
  const size_t N = 65536, B = 1024, bytes = N * B * 8, pitch = B * 8;
  void *h0, *h1, *d0, *d1;
  cudaMallocHost(&h0, bytes); cudaMallocHost(&h1, bytes);
  cudaMalloc(&d0, bytes); cudaMalloc(&d1, bytes);
  cudaStream_t a, b; cudaStreamCreate(&a); cudaStreamCreate(&b);
  cudaEvent_t e0, e1, xa, xb; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventCreate(&xa); cudaEventCreate(&xb);
  auto t = [&](const char* name, auto fn, size_t moved) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0, 0); fn(); cudaEventRecord(e1, 0); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %7.2f ms  %6.1f GB/s\n", name, ms, moved / ms / 1e6);
  };
  auto both = [&](auto h2d, auto d2h) {
    cudaEventRecord(xa, 0); cudaStreamWaitEvent(a, xa); cudaStreamWaitEvent(b, xa);
    h2d(a); d2h(b);
    cudaEventRecord(xa, a); cudaStreamWaitEvent(0, xa);
    cudaEventRecord(xb, b); cudaStreamWaitEvent(0, xb);
  };
  t("H2D 1D 512MiB", [&] { cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, 0); }, bytes);
  t("D2H 1D 512MiB", [&] { cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, 0); }, bytes);
  t("H2D+D2H 1D concurrent", [&] {
    both([&](cudaStream_t s) { cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, s); },
         [&](cudaStream_t s) { cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s); }); }, 2 * bytes);
  for (int C : {2, 4, 8}) {
    const size_t row = pitch / C;
    char nm[64];
    snprintf(nm, sizeof nm, "H2D 2D %dx(%zu B rows)", C, row);
    t(nm, [&] { for (int c = 0; c < C; c++)
        cudaMemcpy2DAsync((char*)d0 + c * N * row, row, (char*)h0 + c * row, pitch, row, N, cudaMemcpyHostToDevice, 0); }, bytes);
    snprintf(nm, sizeof nm, "D2H 2D %dx(%zu B rows)", C, row);
    t(nm, [&] { for (int c = 0; c < C; c++)
        cudaMemcpy2DAsync((char*)h1 + c * row, pitch, (char*)d1 + c * N * row, row, row, N, cudaMemcpyDeviceToHost, 0); }, bytes);
    snprintf(nm, sizeof nm, "H2D+D2H 2D %dx concurrent", C);
    t(nm, [&] {
      both([&](cudaStream_t s) { for (int c = 0; c < C; c++)
             cudaMemcpy2DAsync((char*)d0 + c * N * row, row, (char*)h0 + c * row, pitch, row, N, cudaMemcpyHostToDevice, s); },
           [&](cudaStream_t s) { for (int c = 0; c < C; c++)
             cudaMemcpy2DAsync((char*)h1 + c * row, pitch, (char*)d1 + c * N * row, row, row, N, cudaMemcpyDeviceToHost, s); }); }, 2 * bytes);
  }
  for (int g : {148, 296, 592, 1184}) {
    char nm[64];
    snprintf(nm, sizeof nm, "kernel H2D grid %d", g);
    t(nm, [&] { kcopy<<<g, 512>>>((const int4*)h0, (int4*)d0, bytes / 16); }, bytes);
    snprintf(nm, sizeof nm, "kernel D2H grid %d", g);
    t(nm, [&] { kcopy<<<g, 512>>>((const int4*)d1, (int4*)h1, bytes / 16); }, bytes);
    snprintf(nm, sizeof nm, "kernel H2D+D2H grid %d", g);
    t(nm, [&] { both([&](cudaStream_t s) { kcopy<<<g / 2, 512, 0, s>>>((const int4*)h0, (int4*)d0, bytes / 16); },
                     [&](cudaStream_t s) { kcopy<<<g / 2, 512, 0, s>>>((const int4*)d1, (int4*)h1, bytes / 16); }); }, 2 * bytes);
  }
  return 0;
}
