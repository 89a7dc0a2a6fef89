/* A plain-C consumer of the drop-in boundary (include/b2o.h, libb2o.so): no
 * Python, no torch.  Device buffers come from the CUDA runtime; every result
 * is checked on the host against a C computation of the same operation.
 *
 *   b2o_exact_sum_f32  vs the sequential fp32 loop s = s + x[i]   (bit-exact)
 *   b2o_histogram      vs a host count                            (exact)
 *   b2o_gemm_f32       vs a double-precision host GEMM            (norm-wise 1e-5)
 *
 * Build: make -C tests/c   Run: tests/c/abi_ops   (exit status 0 = pass) */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "b2o.h"

static unsigned long long rng = 20201106ull;
static float urand(void) {
  rng = rng * 6364136223846793005ull + 1442695040888963407ull;
  return (float)((rng >> 40) & 0xFFFFFF) / 16777216.0f;
}

#define CK(x)                                                          \
  do {                                                                 \
    if ((x) != cudaSuccess) {                                          \
      fprintf(stderr, "CUDA error at %s:%d\n", __FILE__, __LINE__);    \
      return 1;                                                        \
    }                                                                  \
  } while (0)

static int exact_sum(void) {
  const int64_t n = 1000003;
  float *h = (float *)malloc(sizeof(float) * n), *d = NULL, *o = NULL, got = 0.f;
  for (int64_t i = 0; i < n; ++i) h[i] = (urand() - 0.25f) * 3.0f;
  volatile float s = 7.5f; /* the loop itself, one fp32 rounding per step */
  for (int64_t i = 0; i < n; ++i) s = s + h[i];
  CK(cudaMalloc((void **)&d, sizeof(float) * n));
  CK(cudaMalloc((void **)&o, sizeof(float)));
  CK(cudaMemcpy(d, h, sizeof(float) * n, cudaMemcpyHostToDevice));
  if (b2o_exact_sum_f32(d, n, 7.5f, o, NULL) != 0) return 1;
  CK(cudaMemcpy(&got, o, sizeof(float), cudaMemcpyDeviceToHost));
  const float want = s;
  printf("exact_sum: got %.9g want %.9g %s\n", got, want, memcmp(&got, &want, 4) == 0 ? "bit-exact" : "DIFFER");
  cudaFree(d);
  cudaFree(o);
  free(h);
  return memcmp(&got, &want, 4) != 0;
}

static int histogram(void) {
  const int64_t n = 1 << 20, bins = 256;
  int32_t *h = (int32_t *)malloc(sizeof(int32_t) * n), *d = NULL, *dh = NULL;
  int32_t want[256] = {0}, got[256];
  for (int64_t i = 0; i < n; ++i) {
    h[i] = (int32_t)(urand() * 300.0f) - 20; /* some out of range: skipped */
    if (h[i] >= 0 && h[i] < bins) want[h[i]]++;
  }
  CK(cudaMalloc((void **)&d, sizeof(int32_t) * n));
  CK(cudaMalloc((void **)&dh, sizeof(int32_t) * bins));
  CK(cudaMemcpy(d, h, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CK(cudaMemset(dh, 0, sizeof(int32_t) * bins));
  if (b2o_histogram(d, n, dh, bins, 0, NULL) != 0) return 1;
  CK(cudaMemcpy(got, dh, sizeof(int32_t) * bins, cudaMemcpyDeviceToHost));
  const int ok = memcmp(got, want, sizeof want) == 0;
  printf("histogram: %s\n", ok ? "exact" : "DIFFER");
  cudaFree(d);
  cudaFree(dh);
  free(h);
  return !ok;
}

static int gemm(void) {
  const int64_t m = 256, n = 256, k = 512;
  float *A = (float *)malloc(sizeof(float) * m * k), *B = (float *)malloc(sizeof(float) * k * n);
  float *C = (float *)malloc(sizeof(float) * m * n), *dA, *dB, *dC;
  for (int64_t i = 0; i < m * k; ++i) A[i] = urand();
  for (int64_t i = 0; i < k * n; ++i) B[i] = urand();
  CK(cudaMalloc((void **)&dA, sizeof(float) * m * k));
  CK(cudaMalloc((void **)&dB, sizeof(float) * k * n));
  CK(cudaMalloc((void **)&dC, sizeof(float) * m * n));
  CK(cudaMemcpy(dA, A, sizeof(float) * m * k, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B, sizeof(float) * k * n, cudaMemcpyHostToDevice));
  if (b2o_gemm_f32(dA, dB, dC, m, n, k, NULL) != 0) return 1;
  CK(cudaMemcpy(C, dC, sizeof(float) * m * n, cudaMemcpyDeviceToHost));
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double r = 0.0;
      for (int64_t p = 0; p < k; ++p) r += (double)A[i * k + p] * (double)B[p * n + j];
      num += (C[i * n + j] - r) * (C[i * n + j] - r);
      den += r * r;
    }
  const double rel = sqrt(num / den);
  printf("gemm (%s path): norm-wise %.3g\n", b2o_gemm_impl() ? "tcgen05 3xTF32" : "SIMT", rel);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  free(A);
  free(B);
  free(C);
  return !(rel < 1e-5);
}

int main(void) {
  printf("b2o ABI %d\n", b2o_abi_version());
  const int rc = exact_sum() | histogram() | gemm();
  printf(rc ? "FAIL\n" : "PASS\n");
  return rc;
}
