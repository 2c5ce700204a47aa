// PCIe bandwidth on the box: 1D / 2D (2 KiB rows) H2D, D2H, and both at once.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t N = 65536, B = 1024, bytes = N * B * 8, row = 256 * 8, pitch = B * 8;
  void *h0, *h1, *d0, *d1;
  cudaMallocHost(&h0, bytes); cudaMallocHost(&h1, bytes);
  cudaMalloc(&d0, bytes); cudaMalloc(&d1, bytes);
  cudaStream_t a, b; cudaStreamCreate(&a); cudaStreamCreate(&b);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto t = [&](const char* name, auto fn, size_t moved) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0, 0); fn(); cudaEventRecord(e1, 0); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %7.2f ms  %6.1f GB/s\n", name, ms, moved / ms / 1e6);
  };
  t("H2D 1D 512MiB", [&] { cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, 0); }, bytes);
  t("D2H 1D 512MiB", [&] { cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, 0); }, bytes);
  t("H2D+D2H 1D concurrent", [&] {
    cudaEventRecord(e0, 0); cudaStreamWaitEvent(a, e0); cudaStreamWaitEvent(b, e0);
    cudaMemcpyAsync(d0, h0, bytes, cudaMemcpyHostToDevice, a);
    cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, b);
    cudaEvent_t x; cudaEventCreate(&x); cudaEventRecord(x, a); cudaStreamWaitEvent(0, x);
    cudaEventRecord(x, b); cudaStreamWaitEvent(0, x); }, 2 * bytes);
  t("H2D 2D 4x(2KiB rows)", [&] { for (int c = 0; c < 4; c++)
      cudaMemcpy2DAsync((char*)d0 + c * N * row, row, (char*)h0 + c * row, pitch, row, N, cudaMemcpyHostToDevice, 0); }, bytes);
  t("D2H 2D 4x(2KiB rows)", [&] { for (int c = 0; c < 4; c++)
      cudaMemcpy2DAsync((char*)h1 + c * row, pitch, (char*)d1 + c * N * row, row, row, N, cudaMemcpyDeviceToHost, 0); }, bytes);
  return 0;
}
