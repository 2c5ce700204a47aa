/* A plain-C client of libfmgsr_cuda.so (no Python, no torch): allocates
 * device memory with the CUDA runtime, builds a plan through the C ABI of
 * include/fmgsr_cuda.h, solves a batch of RHS from host buffers, and prints
 * the worst max-norm relative error against the exact solutions (the
 * discretisation error of one FMG cycle, O(h^2)); exits non-zero above 1e-4
 * or on any ABI error.  Built and run by tests/test_gpu_c_abi.py.
 *
 *   abi_solve m P b B   (fp64, m0 = 3, V(1,1), n_sr = 1)
 */
#include <cuda_runtime.h>
#include <math.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <stdio.h>
#include <stdlib.h>

#include "fmgsr_cuda.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_) {                                                                \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, fmgsr_last_error());     \
      return 2;                                                               \
    }                                                                         \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 5) {
    fprintf(stderr, "usage: abi_solve m P b B\n");
    return 1;
  }
  const int m = atoi(argv[1]);
  const long P = atol(argv[2]), b = atol(argv[3]), B = atol(argv[4]);
  const long n = 1L << m;
  if (fmgsr_abi_version() != FMGSR_ABI_VERSION) return 3;
  /* host forcing: u_r(x) = sin((r + 1) pi x), f_r = ((r + 1) pi)^2 u_r */
  double* hf = (double*)malloc(sizeof(double) * n * B);
  double* hu = (double*)malloc(sizeof(double) * n * B);
  for (long i = 0; i < n; i++)
    for (long r = 0; r < B; r++) {
      const double x = (i + 0.5) / n, k = (double)((r % 4) + 1) * M_PI;
      hf[i * B + r] = k * k * sin(k * x);
    }
  fmgsr_plan_desc d = {0};
  d.m0 = 3;
  d.m = m;
  d.n_sr = 1;
  d.ns = 1;
  d.geom_mode = 2;
  d.dtype = 0;
  d.P = P;
  d.b = b;
  d.B = B;
  d.ld = B;
  d.omega = 1.0;
  d.fused = 1;
  d.use_graph = 1;
  d.coarse = -1;
  d.nonlinear = 0;
  void* plan = NULL;
  CHECK(fmgsr_plan_create(&d, &plan));
  void *df = NULL, *du = NULL;
  if (cudaMalloc(&df, sizeof(double) * n * B) || cudaMalloc(&du, sizeof(double) * n * B)) return 4;
  cudaMemcpy(df, hf, sizeof(double) * n * B, cudaMemcpyHostToDevice);
  CHECK(fmgsr_plan_solve(plan, df, du, NULL));
  if (cudaDeviceSynchronize() != cudaSuccess) return 5;
  cudaMemcpy(hu, du, sizeof(double) * n * B, cudaMemcpyDeviceToHost);
  /* the bad-argument path: a NULL plan is rejected with a message */
  if (fmgsr_plan_solve(NULL, df, du, NULL) != -1 || !fmgsr_last_error()[0]) return 6;
  double worst = 0.0;
  for (long r = 0; r < B; r++) {
    double num = 0.0, den = 0.0;
    for (long i = 0; i < n; i++) {
      const double x = (i + 0.5) / n, k = (double)((r % 4) + 1) * M_PI;
      const double e = hu[i * B + r] - sin(k * x);
      if (fabs(e) > num) num = fabs(e);
      if (fabs(sin(k * x)) > den) den = fabs(sin(k * x));
    }
    if (num / den > worst) worst = num / den;
  }
  printf("abi_solve m=%d P=%ld b=%ld B=%ld max_rel_err=%.3e\n", m, P, b, B, worst);
  CHECK(fmgsr_plan_destroy(plan));
  cudaFree(df);
  cudaFree(du);
  free(hf);
  free(hu);
  return worst < 1e-4 ? 0 : 7;
}
