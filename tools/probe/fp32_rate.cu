// FP32 SIMT issue-rate probe (not product code): FMUL + FADD chains compiled
// with -fmad=false, the operation mix of the exact (uncontracted) loop
// kernels.  8 independent chains per thread hide the 4-cycle latency.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fp32_mul_add(float *out, float a, float b, int iters) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      x[c] = x[c] * a;
      x[c] = x[c] + b;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

__global__ void fp32_fma(float *out, float a, float b, int iters) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = __fmaf_rn(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float *out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 2; ++k) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      if (k == 0) fp32_mul_add<<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      else fp32_fma<<<blocks, threads>>>(out, 0.999f, 1e-4f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    double ops = (double)blocks * threads * iters * 8 * 2;  // 2 flops per chain step
    printf("{\"probe\": \"%s\", \"sms\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n",
           k == 0 ? "fp32_fmul_fadd_no_fma" : "fp32_ffma", sms, best, ops / (best * 1e-3) / 1e12);
  }
  return 0;
}
