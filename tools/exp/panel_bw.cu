// bandwidth of a column-panel read/write pattern: W float2 columns per
// panel-row segment, 4096 rows of 4096 float2 (the FFT column pass access)
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void panel_copy(const float2 *__restrict__ x, float2 *__restrict__ y) {
  // CTA: one panel of W columns, all 4096 rows; 256 threads: row-major over (row, col)
  const int c0 = blockIdx.x * W;
  for (int i = threadIdx.x; i < 4096 * W; i += blockDim.x) {
    const int r = i / W, c = i % W;
    y[(size_t)r * 4096 + c0 + c] = x[(size_t)r * 4096 + c0 + c];
  }
}
int main() {
  float2 *x, *y;
  size_t n = 4096ull * 4096;
  cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8);
  cudaMemset(x, 0, n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
#define RUN(W) { for (int k = 0; k < 3; ++k) panel_copy<W><<<4096 / W, 256>>>(x, y); cudaEventRecord(a); \
  for (int k = 0; k < 10; ++k) panel_copy<W><<<4096 / W, 256>>>(x, y); cudaEventRecord(b); cudaEventSynchronize(b); \
  float ms; cudaEventElapsedTime(&ms, a, b); printf("W=%d segment=%dB: %.1f us, %.0f GB/s\n", W, W * 8, ms * 100, 2.0 * n * 8 / (ms / 10) / 1e6); }
  RUN(4) RUN(8) RUN(16) RUN(32) RUN(64) RUN(128) RUN(256)
  return 0;
}
