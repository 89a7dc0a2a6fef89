// b2o_gemm.cu — the cublas_gemm replacement (reference
// fixtures/sample_db.json:15): C = A B, fp32 row-major.
//
// b2o_gemm_f32 dispatches to the tcgen05/TMEM 3xTF32 kernel in
// b2o_gemm_tc.cu when the shape tiles evenly, else to this SIMT kernel
// (register-tiled FFMA, fp32 accumulation).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/b2o.h"

namespace {

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;

__global__ void __launch_bounds__(256) gemm_simt_kernel(const float *__restrict__ A, const float *__restrict__ B,
                                                        float *__restrict__ C, int M, int N, int K) {
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[TM][TN] = {};
  // each thread loads 4 elements of A (128x8) and 4 of B (8x128) per stage
  auto load = [&](int buf, int k0) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      int r = e / BK, c = e % BK;
      int gm = m0 + r, gk = k0 + c;
      As[buf][c][r] = (gm < M && gk < K) ? A[(size_t)gm * K + gk] : 0.f;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      int r = e / BN, c = e % BN;
      int gk = k0 + r, gn = n0 + c;
      Bs[buf][r][c] = (gk < K && gn < N) ? B[(size_t)gk * N + gn] : 0.f;
    }
  };
  int buf = 0;
  load(0, 0);
  __syncthreads();
  for (int k0 = 0; k0 < K; k0 += BK) {
    if (k0 + BK < K) load(buf ^ 1, k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gn = n0 + tx * TN + j;
      if (gn < N) C[(size_t)gm * N + gn] = acc[i][j];
    }
  }
}

}  // namespace

// provided by b2o_gemm_tc.cu (returns -2 when the shape is not supported)
extern "C" int b2o_gemm_tc_f32(const float *A, const float *B, float *C, int64_t m, int64_t n, int64_t k,
                               void *stream);

extern "C" int b2o_gemm_simt_f32(const float *A, const float *B, float *C, int64_t m, int64_t n, int64_t k,
                                 void *stream) {
  if (m <= 0 || n <= 0 || k <= 0 || m > (1 << 30) || n > (1 << 30) || k > (1 << 30)) return -1;
  dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM));
  gemm_simt_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, B, C, (int)m, (int)n, (int)k);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int b2o_gemm_f32(const float *A, const float *B, float *C, int64_t m, int64_t n, int64_t k,
                            void *stream) {
  int rc = b2o_gemm_tc_f32(A, B, C, m, n, k, stream);
  if (rc != -2) return rc;
  return b2o_gemm_simt_f32(A, B, C, m, n, k, stream);
}

// force-load this file's kernels (lazy module loading would otherwise charge
// the first timed pattern that uses one); called per device by b2o_init
extern "C" void b2o_gemm_warm(void) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, gemm_simt_kernel);
  cudaGetLastError();
}
