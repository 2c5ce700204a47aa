// Dependent-chain latency of fp64 / fp32 ops on the current GPU (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x, double y, int n) {
  double a = x, b = y;
  float fa = (float)x, fb = (float)y;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) { a = __dadd_rn(a, b); }
  long long t1 = clock64();
  for (int i = 0; i < n; i++) { a = __dmul_rn(a, b); }
  long long t2 = clock64();
  for (int i = 0; i < n; i++) { a = __ddiv_rn(a, b); }
  long long t3 = clock64();
  for (int i = 0; i < n; i++) { fa = __fadd_rn(fa, fb); }
  long long t4 = clock64();
  for (int i = 0; i < n; i++) { a = __fma_rn(a, b, y); }
  long long t5 = clock64();
  out[0] = a + fa;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8); cudaMalloc(&c, 64);
  int n = 4096;
  lat<<<1, 1>>>(d, c, 1.0000001, 0.9999999, n);
  lat<<<1, 1>>>(d, c, 1.0000001, 0.9999999, n);
  long long h[5];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[5] = {"DADD", "DMUL", "DDIV(rn)", "FADD", "DFMA"};
  for (int i = 0; i < 5; i++) printf("%-9s %.1f cycles/op (dependent chain)\n", names[i], (double)h[i] / n);
  return 0;
}
