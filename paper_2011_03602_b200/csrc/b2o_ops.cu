// b2o_ops.cu — CPU bindings of opaque library calls and the shared-memory
// FFT that replaces cufft_exec (reference fixtures/sample_db.json:6).
//
// FFT design (HBM-bound): two passes over HBM.
//   n = 4096 (the config-3 size): 4096 = 16 x 16 x 16 four-step factorisation,
//     rows: one CTA per row, first radix-16 pass straight from HBM into
//           registers, last one straight back, two XOR-swizzled shared-memory
//           exchanges in between;
//     cols: in place, one 16-CTA thread-block cluster per 16 adjacent columns
//           (128-byte row segments); the last radix-16 pass gathers across
//           the cluster through distributed shared memory.
//   n = 256: Stockham radix-16 in shared memory; other powers of two: radix-2.
// Twiddles are computed in double on the host and kept in a device table.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/b2o.h"
#include "b2o_module.h"
#include "b2o_ops.h"

namespace cg = cooperative_groups;

// ---------------------------------------------------------------------------
// CPU bindings (the "original library" an unreplaced program calls)
// ---------------------------------------------------------------------------

namespace {

double ld(const void *p, int64_t i, int elem) {
  if (elem == B2O_F64) return ((const double *)p)[i];
  if (elem == B2O_F32) return ((const float *)p)[i];
  return ((const int32_t *)p)[i];
}

void st(void *p, int64_t i, int elem, double v) {
  if (elem == B2O_F64) ((double *)p)[i] = v;
  else if (elem == B2O_F32) ((float *)p)[i] = (float)v;
  else ((int32_t *)p)[i] = (int32_t)v;
}

void fft1d(std::complex<double> *a, int64_t n) {
  if ((n & (n - 1)) != 0) {  // naive DFT for non powers of two
    std::vector<std::complex<double>> out(n);
    for (int64_t k = 0; k < n; ++k) {
      std::complex<double> s = 0;
      for (int64_t t = 0; t < n; ++t) s += a[t] * std::polar(1.0, -2.0 * M_PI * (double)((k * t) % n) / n);
      out[k] = s;
    }
    std::copy(out.begin(), out.end(), a);
    return;
  }
  for (int64_t i = 1, j = 0; i < n; ++i) {
    int64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    for (int64_t i = 0; i < n; i += len) {
      for (int64_t k = 0; k < len / 2; ++k) {
        std::complex<double> w = std::polar(1.0, -2.0 * M_PI * (double)k / (double)len);
        std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
    }
  }
}

}  // namespace

extern "C" void b2o_cpu_gemm(const void *A, const void *B, void *C, int64_t m, int64_t n, int64_t k, int elem) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    std::vector<double> acc(n, 0.0);
    for (int64_t kk = 0; kk < k; ++kk) {
      double a = ld(A, i * k + kk, elem);
      const int64_t base = kk * n;
      if (elem == B2O_F32) {
        const float *b = (const float *)B + base;
        for (int64_t j = 0; j < n; ++j) acc[j] += a * (double)b[j];
      } else {
        for (int64_t j = 0; j < n; ++j) acc[j] += a * ld(B, base + j, elem);
      }
    }
    for (int64_t j = 0; j < n; ++j) st(C, i * n + j, elem, acc[j]);
  }
}

extern "C" void b2o_cpu_fft2d(const void *x, void *y, int64_t n, int elem) {
  std::vector<std::complex<double>> a((size_t)(n * n));
  for (int64_t i = 0; i < n * n; ++i) a[i] = {ld(x, 2 * i, elem), ld(x, 2 * i + 1, elem)};
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) fft1d(&a[r * n], n);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    std::vector<std::complex<double>> col(n);
    for (int64_t r = 0; r < n; ++r) col[r] = a[r * n + c];
    fft1d(col.data(), n);
    for (int64_t r = 0; r < n; ++r) a[r * n + c] = col[r];
  }
  for (int64_t i = 0; i < n * n; ++i) {
    st(y, 2 * i, elem, a[i].real());
    st(y, 2 * i + 1, elem, a[i].imag());
  }
}

extern "C" void b2o_cpu_histogram(const int32_t *d, int64_t n, void *h, int64_t bins, int elem) {
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b = d[i];
    if (b < 0 || b >= bins) continue;
    if (elem == B2O_I32) ((int32_t *)h)[b] += 1;
    else if (elem == B2O_F32) ((float *)h)[b] += 1.0f;
    else ((double *)h)[b] += 1.0;
  }
}

// ---------------------------------------------------------------------------
// GPU histogram (cuda_histogram replacement, fixtures/sample_db.json:20-28)
//
// HBM-bound: 4 B read per element.  16-byte vector loads, grid sized to the
// 148 SMs; counts go to per-warp private copies of the histogram in shared
// memory when bins x warps fit (no cross-warp contention on skewed data),
// else to one shared copy per CTA, else straight to global atomics; each
// CTA then adds its non-zero bins to h with one atomic per bin.  Integer
// counts make the result exact and order-independent (bit-exact to the
// sequential loop; float h exact below 2^24 per bin).
// ---------------------------------------------------------------------------

namespace {

constexpr int kHistThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kHistThreads) hist_smem_kernel(const int32_t *__restrict__ d, int64_t n,
                                                                  T *__restrict__ h, int bins, int copies) {
  extern __shared__ uint32_t sh[];  // copies x bins
  const int total = copies * bins;
  for (int i = threadIdx.x; i < total; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t *mine = sh + (copies > 1 ? (threadIdx.x / 32) % copies : 0) * bins;
  const uint32_t ub = (uint32_t)bins;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = (((uintptr_t)d & 15) == 0) ? n / 4 : 0;
  const int4 *d4 = (const int4 *)d;
  auto count4 = [&](const int4 q) {
    if ((uint32_t)q.x < ub) atomicAdd(&mine[q.x], 1u);
    if ((uint32_t)q.y < ub) atomicAdd(&mine[q.y], 1u);
    if ((uint32_t)q.z < ub) atomicAdd(&mine[q.z], 1u);
    if ((uint32_t)q.w < ub) atomicAdd(&mine[q.w], 1u);
  };
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // four independent 16-byte loads in flight per thread before the atomics
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const int4 q0 = __ldcs(d4 + i), q1 = __ldcs(d4 + i + stride), q2 = __ldcs(d4 + i + 2 * stride),
               q3 = __ldcs(d4 + i + 3 * stride);  // streamed once: evict-first
    count4(q0);
    count4(q1);
    count4(q2);
    count4(q3);
  }
  for (; i < n4; i += stride) count4(__ldcs(d4 + i));
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t v = d[i];
    if ((uint32_t)v < ub) atomicAdd(&mine[v], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x) {
    uint32_t c = 0;
    for (int k = 0; k < copies; ++k) c += sh[k * bins + b];
    if (c) atomicAdd(&h[b], (T)c);
  }
}

template <typename T>
__global__ void __launch_bounds__(kHistThreads) hist_global_kernel(const int32_t *__restrict__ d, int64_t n,
                                                                    T *__restrict__ h, int64_t bins) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t v = d[i];
    if (v >= 0 && v < bins) atomicAdd(&h[v], (T)1);
  }
}

template <typename T>
int launch_hist(const int32_t *d, int64_t n, T *h, int64_t bins, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t smem_cap = 96 * 1024;  // at least two CTAs per SM
  if (bins * 4 <= smem_cap) {
    const int warps = kHistThreads / 32;
    int copies = (int)std::min<int64_t>(warps, smem_cap / (bins * 4));
    while (copies > 1 && warps % copies) --copies;
    const size_t smem = (size_t)copies * bins * 4;
    cudaFuncSetAttribute(hist_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap);
    const int64_t want = (n / 4 + kHistThreads - 1) / kHistThreads;
    // three CTAs per SM when their private copies fit (64 M int32, 256 bins:
    // 48.1 -> 44.0 us, 0.85 -> 0.93 of HBM; four: 44.6 us)
    static const int env_per_sm = getenv("B2O_HIST_CTAS") ? atoi(getenv("B2O_HIST_CTAS")) : 0;
    const int per_sm = env_per_sm > 0 ? env_per_sm : (smem <= 72 * 1024 ? 3 : 2);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));
    hist_smem_kernel<T><<<grid, kHistThreads, smem, s>>>(d, n, h, (int)bins, copies);
  } else {
    const int64_t want = (n + kHistThreads - 1) / kHistThreads;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 4));
    hist_global_kernel<T><<<grid, kHistThreads, 0, s>>>(d, n, h, bins);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

extern "C" int b2o_histogram(const int32_t *d, int64_t n, void *h, int64_t bins, int elem, void *stream) {
  if (n < 0 || bins <= 0) return -1;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (elem == B2O_I32) return launch_hist<int32_t>(d, n, (int32_t *)h, bins, s);
  if (elem == B2O_F32) return launch_hist<float>(d, n, (float *)h, bins, s);
  if (elem == B2O_F64) return launch_hist<double>(d, n, (double *)h, bins, s);
  return -1;
}

// ---------------------------------------------------------------------------
// GPU FFT
// ---------------------------------------------------------------------------

namespace {

constexpr int kFftThreads = 512;
constexpr int kColGroup = 4;

// in-place radix-2 DIT over `count` independent length-n sequences stored
// back to back in shared memory, already in bit-reversed order
__device__ __forceinline__ void smem_fft(float2 *s, int n, int logn, int count, const float2 *__restrict__ tw) {
  const int half = n >> 1;
  for (int st = 0; st < logn; ++st) {
    const int span = 1 << st;        // butterfly half-width
    const int tw_shift = logn - 1 - st;  // twiddle index = k * n / (2*span)
    for (int b = threadIdx.x; b < half * count; b += blockDim.x) {
      const int seq = b / half;
      const int bb = b - seq * half;
      const int k = bb & (span - 1);
      const int i0 = ((bb >> st) << (st + 1)) + k;
      float2 *base = s + seq * n;
      const float2 w = tw[k << tw_shift];
      const float2 u = base[i0];
      const float2 v0 = base[i0 + span];
      const float2 v = make_float2(v0.x * w.x - v0.y * w.y, v0.x * w.y + v0.y * w.x);
      base[i0] = make_float2(u.x + v.x, u.y + v.y);
      base[i0 + span] = make_float2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kFftThreads) fft_rows_kernel(const float2 *__restrict__ x, float2 *__restrict__ y,
                                                              int n, int logn, const float2 *__restrict__ tw) {
  extern __shared__ float2 s[];
  const size_t row = blockIdx.x;
  const float2 *src = x + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[__brev(i) >> (32 - logn)] = src[i];
  __syncthreads();
  smem_fft(s, n, logn, 1, tw);
  float2 *dst = y + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = s[i];
}

__global__ void __launch_bounds__(kFftThreads) fft_cols_kernel(float2 *__restrict__ y, int n, int logn,
                                                              const float2 *__restrict__ tw) {
  extern __shared__ float2 s[];
  const int c0 = blockIdx.x * kColGroup;
  for (int idx = threadIdx.x; idx < n * kColGroup; idx += blockDim.x) {
    const int r = idx / kColGroup, c = idx - r * kColGroup;
    s[c * n + (__brev(r) >> (32 - logn))] = y[(size_t)r * n + c0 + c];
  }
  __syncthreads();
  smem_fft(s, n, logn, kColGroup, tw);
  for (int idx = threadIdx.x; idx < n * kColGroup; idx += blockDim.x) {
    const int r = idx / kColGroup, c = idx - r * kColGroup;
    y[(size_t)r * n + c0 + c] = s[c * n + r];
  }
}

// ---- radix-16 path (N = 16^P): digit-reversed load, in-place DIT passes,
// each thread owns whole 16-point groups in registers ----------------------

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// 16-point DFT of v[0..15] in registers (natural order in, natural order out)
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
  // radix-2 DIF stages with the 16th roots of unity, then bit-reverse
  const float c1 = 0.92387953251128674f, s1 = 0.38268343236508978f, r2 = 0.70710678118654752f;
  const float2 w[8] = {{1.f, 0.f}, {c1, -s1}, {r2, -r2}, {s1, -c1}, {0.f, -1.f}, {-s1, -c1}, {-r2, -r2}, {-c1, -s1}};
#pragma unroll
  for (int span = 8, step = 1; span >= 1; span >>= 1, step <<= 1) {
#pragma unroll
    for (int base = 0; base < 16; base += 2 * span) {
#pragma unroll
      for (int k = 0; k < span; ++k) {
        float2 a = v[base + k], b = v[base + k + span];
        v[base + k] = make_float2(a.x + b.x, a.y + b.y);
        v[base + k + span] = cmul(make_float2(a.x - b.x, a.y - b.y), w[k * step]);
      }
    }
  }
  // outputs are bit-reversed: swap into natural order
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = ((i & 1) << 3) | ((i & 2) << 1) | ((i & 4) >> 1) | ((i & 8) >> 3);
    if (r > i) {
      float2 t = v[i];
      v[i] = v[r];
      v[r] = t;
    }
  }
}

// shared-memory swizzle: XOR the low nibble of the float2 index with the
// next nibble, so every pass of the Stockham radix-16 FFT below (reads at
// stride N/16, writes at stride L, plus the natural-order load/store) hits 16
// distinct 8-byte bank pairs per half-warp
__device__ __forceinline__ int sw16(int i) { return i ^ ((i >> 4) & 15); }

// Stockham autosort radix-16 FFT (natural order in and out) over COUNT
// sequences of length n = 16^digits, interleaved in shared memory: element i
// of sequence c lives at s[sw16(i) * COUNT + c] (so COUNT adjacent columns of
// a matrix are stored the way they arrive from global memory).  Each pass
// reads a thread's 16-point groups into registers, barrier, writes them back:
// in place without a second buffer.  Consecutive threads take consecutive
// sequences of the same group (conflict-free), twiddles come from one table
// load per group and a complex recurrence.  tw[m] = exp(-2 pi i m / n).
template <int COUNT, int GROUPS_PER_THREAD>
__device__ void smem_fft16(float2 *s, int n, int digits, const float2 *__restrict__ tw) {
  const int stride_in = n / 16;
  for (int p = 0, L = 1; p < digits; ++p, L *= 16) {
    const int tw_scale = n / (16 * L);
    float2 v[GROUPS_PER_THREAD][16];
    int dst[GROUPS_PER_THREAD];
#pragma unroll
    for (int q = 0; q < GROUPS_PER_THREAD; ++q) {
      const int g = threadIdx.x + q * blockDim.x;
      const int c = g % COUNT;
      const int gg = g / COUNT;  // = j * L + k
      const int k = gg % L;
      const int j = gg / L;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[q][r] = s[sw16(gg + r * stride_in) * COUNT + c];
      if (p > 0 && k > 0) {
        const float2 w1 = tw[(k * tw_scale) & (n - 1)];
        float2 w = w1;
#pragma unroll
        for (int r = 1; r < 16; ++r) {
          v[q][r] = cmul(v[q][r], w);
          w = cmul(w, w1);
        }
      }
      dft16(v[q]);
      dst[q] = (j * 16 * L + k) * COUNT + c;  // element index * COUNT + c, before swizzle
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GROUPS_PER_THREAD; ++q) {
      const int c = dst[q] % COUNT;
      const int e = dst[q] / COUNT;
#pragma unroll
      for (int r = 0; r < 16; ++r) s[sw16(e + r * L) * COUNT + c] = v[q][r];
    }
    __syncthreads();
  }
}

constexpr int kColGroup16 = 2;  // 2 columns (64 KB smem): 3 CTAs per SM overlap load/compute/store

__global__ void __launch_bounds__(256) fft16_rows_kernel(const float2 *__restrict__ x, float2 *__restrict__ y, int n,
                                                         int digits, const float2 *__restrict__ tw) {
  extern __shared__ float2 s[];
  const size_t row = blockIdx.x;
  const float2 *src = x + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[sw16(i)] = src[i];
  __syncthreads();
  smem_fft16<1, 1>(s, n, digits, tw);
  float2 *dst = y + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = s[sw16(i)];
}

__global__ void __launch_bounds__(512, 2) fft16_cols_kernel(float2 *__restrict__ y, int n, int digits,
                                                         const float2 *__restrict__ tw) {
  extern __shared__ float2 s[];
  const int c0 = blockIdx.x * kColGroup16;
  for (int idx = threadIdx.x; idx < n * kColGroup16; idx += blockDim.x) {
    const int r = idx / kColGroup16, c = idx - r * kColGroup16;
    s[sw16(r) * kColGroup16 + c] = y[(size_t)r * n + c0 + c];
  }
  __syncthreads();
  smem_fft16<kColGroup16, 1>(s, n, digits, tw);
  for (int idx = threadIdx.x; idx < n * kColGroup16; idx += blockDim.x) {
    const int r = idx / kColGroup16, c = idx - r * kColGroup16;
    y[(size_t)r * n + c0 + c] = s[sw16(r) * kColGroup16 + c];
  }
}

// ---- 4096-point path: 4096 = 16 x 16 x 16 as a four-step factorisation
//   n = n2 + 16 (b + 16 a),  k = k1a + 16 k1b + 256 k2
//   X[k] = sum_n2 W16^(n2 k2) W4096^(n2 k1) sum_b W16^(b k1b) W256^(b k1a) sum_a W16^(a k1a) x[n]
// pass 1 (DFT over a) reads HBM straight into registers, pass 3 (DFT over
// n2) stores straight to HBM, so a 4096-point FFT costs two shared-memory
// exchanges (XOR-swizzled: conflict-free) instead of four.

// rows: one CTA (256 threads, 32 KB smem) per 4096-point row
__global__ void __launch_bounds__(256) fft4k_rows_kernel(const float2 *__restrict__ x, float2 *__restrict__ y,
                                                          const float2 *__restrict__ tw) {
  __shared__ float2 s[4096];
  // the column pass (programmatic dependent launch) may start launching now;
  // it waits for this grid's completion before reading y
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int t = threadIdx.x;
  const float2 *src = x + (size_t)blockIdx.x * 4096;
  float2 v[16];
  // pass 1: thread (n2 = t & 15, b = t >> 4) owns n = t + 256 a
#pragma unroll
  for (int a = 0; a < 16; ++a) v[a] = src[t + 256 * a];
  dft16(v);
  {
    const int n2 = t & 15, b = t >> 4;
    const float2 w1 = tw[16 * b];
    float2 w = w1;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      v[k] = cmul(v[k], w);
      w = cmul(w, w1);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) s[n2 * 256 + k * 16 + (b ^ n2)] = v[k];
  }
  __syncthreads();
  // pass 2: thread (n2 = t & 15, k1a = t >> 4), DFT over b
  {
    const int n2 = t & 15, k1a = t >> 4;
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = s[n2 * 256 + k1a * 16 + (b ^ n2)];
    __syncthreads();
    dft16(v);
    const float2 step = tw[16 * n2];
    float2 w = tw[n2 * k1a];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = cmul(v[k], w);
      w = cmul(w, step);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) s[(k1a + 16 * k) * 16 + (n2 ^ k1a)] = v[k];
  }
  __syncthreads();
  // pass 3: thread k1 = t, DFT over n2, coalesced stores X[k1 + 256 k2]
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = s[t * 16 + (n2 ^ (t & 15))];
  dft16(v);
  float2 *dst = y + (size_t)blockIdx.x * 4096;
#pragma unroll
  for (int k = 0; k < 16; ++k) dst[t + 256 * k] = v[k];
}

// columns, in place: a thread-block CLUSTER of kClusterFft CTAs owns 16
// adjacent columns (128-byte row segments: full sectors, one HBM read and one
// write of every element).  CTA rank c holds the 256-point sub-FFTs of the
// rows n2 = c*NPC .. (c+1)*NPC-1 (mod 16) in its shared memory; the final DFT
// over n2 gathers its 16 inputs from the peer CTAs through distributed
// shared memory (ld.shared::cluster), so the 4096-point column FFT never
// round-trips through HBM.
constexpr int kClusterFft = 16;

template <int NPC, int V>
__global__ void __launch_bounds__(256 * NPC, V == 2 ? 6 / NPC : V == 3 ? 5 / NPC : 0)
    fft4k_cols_cluster_kernel(float2 *__restrict__ y, const float2 *__restrict__ tw) {
  extern __shared__ float2 s[];  // NPC x 4096
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the rows pass has completed and is visible
  cg::cluster_group cl = cg::this_cluster();
  constexpr int CL = 16 / NPC;
  const int c = (int)cl.block_rank();
  const int col0 = (int)(blockIdx.x / CL) * 16;
  const int t = threadIdx.x & 255, sub = threadIdx.x >> 8;
  const int n2 = c * NPC + sub;
  float2 *sz = s + sub * 4096;
  const int cc = t & 15;
  float2 v[16];
  {
    const int b = t >> 4;
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = y[(size_t)(n2 + 16 * (b + 16 * a)) * 4096 + col0 + cc];
    dft16(v);
    const float2 w1 = tw[16 * b];
    float2 w = w1;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      v[k] = cmul(v[k], w);
      w = cmul(w, w1);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) sz[(b * 16 + k) * 16 + cc] = v[k];
  }
  __syncthreads();
  {
    const int k1a = t >> 4;
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = sz[(b * 16 + k1a) * 16 + cc];
    __syncthreads();
    dft16(v);
    const float2 step = tw[16 * n2];
    float2 w = tw[n2 * k1a];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = cmul(v[k], w);
      w = cmul(w, step);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) sz[(k1a + 16 * k) * 16 + cc] = v[k];
  }
  // every CTA's Y[k1][cc] is published to the cluster
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  {
    const int k1 = c * 16 * NPC + (threadIdx.x >> 4);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const float2 *peer = cl.map_shared_rank(s, m / NPC) + (m % NPC) * 4096;
      v[m] = peer[k1 * 16 + cc];
    }
    dft16(v);
    // done reading peers; the wait at the end keeps this CTA's shared
    // memory alive until every peer has read it, overlapping the HBM stores.
    // V >= 1: a relaxed arrive -- the peer values were consumed by the DFT
    // above, so the remote loads have completed and need no release fence
    if (V >= 1)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    else
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 16; ++k) y[(size_t)(k1 + 256 * k) * 4096 + col0 + cc] = v[k];
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

template <int NPC, int V = 1>
cudaError_t launch_cols_cluster(float2 *y, const float2 *tw, cudaStream_t s) {
  static const int v_env = getenv("B2O_FFT_V") ? atoi(getenv("B2O_FFT_V")) : -1;
  if (V == 1 && v_env == 0) return launch_cols_cluster<NPC, 0>(y, tw, s);
  if (V == 1 && v_env == 2) return launch_cols_cluster<NPC, 2>(y, tw, s);
  if (V == 1 && v_env == 3) return launch_cols_cluster<NPC, 3>(y, tw, s);
  constexpr int CL = 16 / NPC;
  auto kern = fft4k_cols_cluster_kernel<NPC, V>;
  const size_t smem = sizeof(float2) * 4096 * NPC;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((4096 / 16) * CL);
  cfg.blockDim = dim3(256 * NPC);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = getenv("B2O_PDL") && atoi(getenv("B2O_PDL")) == 0 ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, y, tw);
}

// ---- persistent, TMA-fed column pass (opt-in, B2O_FFT_COLS=persist) ---------
// The cluster kernel above is one load -> compute -> exchange -> store phase
// per CTA, 4096 short-lived CTAs in 16-CTA clusters: every CTA waits for its
// own loads and then for the cluster barrier, with little else resident to
// overlap them (ncu: DRAM 29 % busy, barrier + membar + long-scoreboard
// stalls).  Here 18 clusters stay resident (2 CTAs per SM, 96 KB smem each)
// and walk the 256 column groups: CTA rank c's 256 x 16 slice of the next
// group (rows c + 16 m, one 128-byte segment per row) is fetched by ONE
// 3-D TMA copy into its input buffer as soon as the current group's first
// radix-16 pass has read it, so the HBM reads of group g+1 run under the
// DFTs, the cluster exchange and the stores of group g.  The exchange buffer
// is double-buffered across groups, so one cluster barrier per group suffices
// (a CTA passing the barrier of group g+1 knows every peer finished reading
// its exchange buffer of group g).
namespace colp {

constexpr int IN_BYTES = 256 * 16 * 8;   // 32 KB: rows c + 16 m, 16 columns
constexpr int SZ_ELEMS = 4096;           // 32 KB exchange buffer (x2)
constexpr int SMEM = IN_BYTES + 2 * SZ_ELEMS * 8 + 64;

__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(b)
      : "memory");
}

__global__ void __launch_bounds__(256, 2) fft4k_cols_persist_kernel(float2 *__restrict__ y,
                                                                     const float2 *__restrict__ tw,
                                                                     const __grid_constant__ CUtensorMap map,
                                                                     int nclusters) {
  extern __shared__ __align__(128) uint8_t sm[];
  float2 *in = (float2 *)sm;                             // [m][cc]
  float2 *szb = (float2 *)(sm + IN_BYTES);               // [2][4096]
  uint64_t *bar = (uint64_t *)(sm + IN_BYTES + 2 * SZ_ELEMS * 8);
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();                    // residue class n2 = c
  const int cid = (int)(blockIdx.x / 16);
  const int t = threadIdx.x, cc = t & 15, b = t >> 4;
  const uint32_t inb = su32(in), barb = su32(bar);
  if (t == 0) {
    bar_init(barb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map) : "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the rows pass has completed and is visible
  if (t == 0 && cid < 256) {
    bar_expect(barb, IN_BYTES);
    tma3(inb, &map, 32 * cid, c, 0, barb);
  }
  float2 v[16];
  int g = 0;
  for (int p = cid; p < 256; p += nclusters, ++g) {
    float2 *sz = szb + (g & 1) * SZ_ELEMS;
    const int col0 = p * 16;
    bar_wait(barb, g & 1);
    // pass 1 (DFT over a) from the TMA-landed slice: x[n2 + 16 (b + 16 a)]
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = in[(b + 16 * a) * 16 + cc];
    __syncthreads();  // the slice is consumed: fetch the next group's
    if (t == 0 && p + nclusters < 256) {
      bar_expect(barb, IN_BYTES);
      tma3(inb, &map, 32 * (p + nclusters), c, 0, barb);
    }
    dft16(v);
    {
      const float2 w1 = tw[16 * b];
      float2 w = w1;
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        v[k] = cmul(v[k], w);
        w = cmul(w, w1);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) sz[(b * 16 + k) * 16 + cc] = v[k];
    }
    __syncthreads();
    {
      const int k1a = t >> 4;
#pragma unroll
      for (int bb = 0; bb < 16; ++bb) v[bb] = sz[(bb * 16 + k1a) * 16 + cc];
      __syncthreads();
      dft16(v);
      const float2 step = tw[16 * c];
      float2 w = tw[c * k1a];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        v[k] = cmul(v[k], w);
        w = cmul(w, step);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) sz[(k1a + 16 * k) * 16 + cc] = v[k];
    }
    // publish this group's Y[k1][cc]; passing it also means every peer has
    // finished reading the other exchange buffer (group g-1)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    {
      const int k1 = c * 16 + (t >> 4);
#pragma unroll
      for (int m = 0; m < 16; ++m) v[m] = cl.map_shared_rank(sz, m)[k1 * 16 + cc];
      dft16(v);
#pragma unroll
      for (int k = 0; k < 16; ++k) y[(size_t)(k1 + 256 * k) * 4096 + col0 + cc] = v[k];
    }
  }
  // keep the exchange buffers alive until every peer has read them
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess)
      fn = (EncodeFn)q;
  });
  return fn;
}

// the 4096 x 4096 complex64 matrix as a 3-D fp32 tensor: (32 floats = 16
// complex columns, residue class n2 of the row, row block m), box {32, 1, 256}
cudaError_t launch(float2 *y, const float2 *tw, cudaStream_t s, int nclusters) {
  EncodeFn enc = encode();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[3] = {8192, 16, 256};
  cuuint64_t strides[2] = {8192 * 4, 16 * 8192 * 4};
  cuuint32_t box[3] = {32, 1, 256};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)y, dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  cudaFuncSetAttribute(fft4k_cols_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(fft4k_cols_persist_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(16 * nclusters));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = getenv("B2O_PDL") && atoi(getenv("B2O_PDL")) == 0 ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fft4k_cols_persist_kernel, y, tw, map, nclusters);
}

// clusters of 16 that fit at once (the occupancy calculator for this exact
// configuration), capped at the 256 column groups
int max_clusters(float2 *y, const float2 *tw) {
  cudaFuncSetAttribute(fft4k_cols_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(fft4k_cols_persist_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16 * 64);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (const void *)fft4k_cols_persist_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(n, 256);
}

}  // namespace colp

std::mutex tw_mu;
std::map<std::pair<int, int64_t>, float2 *> tw_cache;  // (device, n) -> table
// per-device "dynamic shared memory attribute set" flags (cleared when the
// runtime resets a device, b2o_ops_forget_device)
std::atomic<bool> g_attr16[64], g_attr_set[64];

float2 *twiddles(int64_t n, bool full = false) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(tw_mu);
  auto key = std::make_pair(dev, full ? -n : n);
  auto it = tw_cache.find(key);
  if (it != tw_cache.end()) return it->second;
  std::vector<float2> h(full ? n : n / 2);
  for (int64_t k = 0; k < (int64_t)h.size(); ++k) {
    double a = -2.0 * M_PI * (double)k / (double)n;
    h[k] = make_float2((float)cos(a), (float)sin(a));
  }
  float2 *d = nullptr;
  if (cudaMalloc(&d, sizeof(float2) * h.size()) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice);
  tw_cache[key] = d;
  return d;
}

}  // namespace

extern "C" int b2o_fft2d_c64(const float *x, float *y, int64_t n, void *stream) {
  if (n < 8 || n > 4096 || (n & (n - 1)) != 0 || n % kColGroup != 0) return -1;
  int digits16 = 0;
  for (int64_t m = 1; m < n; m *= 16) ++digits16;
  if ((int64_t)1 << (4 * digits16) == n && n >= 256) {
    float2 *tw = twiddles(n, true);
    if (!tw) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    std::atomic<bool> *attr16 = g_attr16;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr16[dev & 63]) {
      cudaFuncSetAttribute(fft16_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(fft16_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr16[dev & 63] = true;
    }
    if (n == 4096 && !getenv("B2O_FFT_LEGACY")) {
      fft4k_rows_kernel<<<4096, 256, 0, s>>>((const float2 *)x, (float2 *)y, tw);
      // B2O_FFT_COLS=persist: the persistent TMA-fed column pass (measured
      // slower: 0.157 vs 0.126 ms -- 14 resident clusters leave 21 % of the
      // warps active, too few to hide the per-group barrier and DSMEM
      // latency that 5 short-lived CTAs per SM overlap); default: the
      // per-group cluster kernel below
      static std::atomic<int> ncl[64];
      static const bool old_cols = !(getenv("B2O_FFT_COLS") && std::string(getenv("B2O_FFT_COLS")) == "persist");
      if (!old_cols && ncl[dev & 63] == 0) {
        int m = colp::max_clusters((float2 *)y, tw);
        if (getenv("B2O_FFT_CLUSTERS")) m = std::min(m, atoi(getenv("B2O_FFT_CLUSTERS")));
        ncl[dev & 63] = m > 0 ? m : -1;
      }
      if (!old_cols && ncl[dev & 63] > 0) {
        if (colp::launch((float2 *)y, tw, s, ncl[dev & 63]) == cudaSuccess)
          return cudaGetLastError() == cudaSuccess ? 0 : -1;
        cudaGetLastError();
        ncl[dev & 63] = -1;  // nothing ran: the cluster kernel below instead
      }
      // cluster of 16 CTAs (non-portable size) when the device takes it, else 8 x 2 sub-FFTs
      static std::atomic<int> npc[64];
      if (npc[dev & 63] == 0 && getenv("B2O_FFT_NPC")) npc[dev & 63] = atoi(getenv("B2O_FFT_NPC"));
      if (npc[dev & 63] == 0) {
        cudaError_t e = launch_cols_cluster<1>((float2 *)y, tw, s);
        if (e == cudaSuccess) {
          npc[dev & 63] = 1;
        } else {
          cudaGetLastError();
          npc[dev & 63] = 2;
          // the 16-CTA cluster did not launch (nothing ran): use 8 CTAs x 2 sub-FFTs
          if (launch_cols_cluster<2>((float2 *)y, tw, s) != cudaSuccess) return -1;
        }
      } else if (npc[dev & 63] == 1) {
        if (launch_cols_cluster<1>((float2 *)y, tw, s) != cudaSuccess) return -1;
      } else {
        if (launch_cols_cluster<2>((float2 *)y, tw, s) != cudaSuccess) return -1;
      }
      return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    if (n != 4096 && n != 256) return -1;
    fft16_rows_kernel<<<(unsigned)n, (unsigned)(n / 16), sizeof(float2) * n, s>>>((const float2 *)x, (float2 *)y,
                                                                             (int)n, digits16, tw);
    fft16_cols_kernel<<<(unsigned)(n / kColGroup16), (unsigned)(n / 16 * kColGroup16), sizeof(float2) * n * kColGroup16, s>>>(
        (float2 *)y, (int)n, digits16, tw);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
  }
  int logn = 0;
  while ((1 << logn) < n) ++logn;
  float2 *tw = twiddles(n);
  if (!tw) return -1;
  cudaStream_t s = (cudaStream_t)stream;
  size_t row_smem = sizeof(float2) * n;
  size_t col_smem = sizeof(float2) * n * kColGroup;
  std::atomic<bool> *attr_set = g_attr_set;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(fft_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fft_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set[dev & 63] = true;
  }
  fft_rows_kernel<<<(unsigned)n, kFftThreads, row_smem, s>>>((const float2 *)x, (float2 *)y, (int)n, logn, tw);
  fft_cols_kernel<<<(unsigned)(n / kColGroup), kFftThreads, col_smem, s>>>((float2 *)y, (int)n, logn, tw);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// the device was reset (runtime broken-worker recovery): its twiddle tables
// and function attributes are gone with the context
extern "C" void b2o_ops_forget_device(int dev) {
  std::lock_guard<std::mutex> lk(tw_mu);
  for (auto it = tw_cache.begin(); it != tw_cache.end();) {
    if (it->first.first == dev) it = tw_cache.erase(it);
    else ++it;
  }
  g_attr16[dev & 63] = false;
  g_attr_set[dev & 63] = false;
}

// force-load this file's kernels (lazy module loading would otherwise charge
// the first timed pattern that uses one); called per device by b2o_init
extern "C" void b2o_ops_warm(void) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void *)hist_smem_kernel<int32_t>);
  cudaFuncGetAttributes(&a, (const void *)hist_smem_kernel<float>);
  cudaFuncGetAttributes(&a, (const void *)hist_smem_kernel<double>);
  cudaFuncGetAttributes(&a, (const void *)hist_global_kernel<int32_t>);
  cudaFuncGetAttributes(&a, (const void *)hist_global_kernel<float>);
  cudaFuncGetAttributes(&a, (const void *)hist_global_kernel<double>);
  cudaFuncGetAttributes(&a, fft_rows_kernel);
  cudaFuncGetAttributes(&a, fft_cols_kernel);
  cudaFuncGetAttributes(&a, fft16_rows_kernel);
  cudaFuncGetAttributes(&a, fft16_cols_kernel);
  cudaFuncGetAttributes(&a, fft4k_rows_kernel);
  cudaFuncGetAttributes(&a, (const void *)fft4k_cols_cluster_kernel<1, 1>);
  cudaFuncGetAttributes(&a, (const void *)colp::fft4k_cols_persist_kernel);
  cudaFuncGetAttributes(&a, (const void *)fft4k_cols_cluster_kernel<2, 1>);
  cudaGetLastError();
}
