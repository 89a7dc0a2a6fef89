// Output comparison on the device (the measurement's validate_output step,
// reference src/evaluators.py:129-139): an output the run left valid in HBM
// is checked against a device copy of the reference output instead of being
// downloaded and compared on the host.  Same rule, same arithmetic (double,
// no contraction), so the verdict, the mismatch count and the worst relative
// error equal the host comparison (b2o_runtime.cu compare_elementwise); the
// norm-wise variant sums per-CTA partials in a fixed order (deterministic).
//
// HBM-bound: reads candidate + reference once (8 B per fp32 element).

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "b2o_module.h"
#include "b2o_ops.h"

namespace {

constexpr int kThreads = 256;
constexpr int kBlocksPerSm = 8;

struct CmpAcc {
  unsigned long long bad;
  unsigned long long worst_bits;  // max over non-negative doubles: integer order == value order
  int nan;
  int pad;
  double part[1];                 // norm-wise: 2 doubles per CTA (num, den)
};

template <typename T>
__device__ __forceinline__ void cmp_one(T c, T r, double tol, unsigned long long &bad, double &worst, int &nan) {
  if (c == r) return;  // the common, bit-exact case
  const double cd = (double)c, rd = (double)r;
  const double diff = fabs(cd - rd);
  const double ar = fabs(rd);
  bad += !(diff <= fmax(tol * ar, 1e-12));
  const double rel = diff / fmax(ar, 1e-30);
  nan |= rel != rel;
  worst = rel > worst ? rel : worst;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) cmp_elem_kernel(const T *__restrict__ cand, const T *__restrict__ ref,
                                                            int64_t n, double tol, CmpAcc *acc) {
  unsigned long long bad = 0;
  double worst = 0.0;
  int nan = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    T c0 = cand[i], c1 = cand[i + stride], c2 = cand[i + 2 * stride], c3 = cand[i + 3 * stride];
    T r0 = ref[i], r1 = ref[i + stride], r2 = ref[i + 2 * stride], r3 = ref[i + 3 * stride];
    cmp_one(c0, r0, tol, bad, worst, nan);
    cmp_one(c1, r1, tol, bad, worst, nan);
    cmp_one(c2, r2, tol, bad, worst, nan);
    cmp_one(c3, r3, tol, bad, worst, nan);
  }
  for (; i < n; i += stride) cmp_one(cand[i], ref[i], tol, bad, worst, nan);
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
  if ((threadIdx.x & 31) == 0 && (bad || worst > 0.0 || nan)) {
    if (bad) atomicAdd(&acc->bad, bad);
    if (worst > 0.0) atomicMax(&acc->worst_bits, (unsigned long long)__double_as_longlong(worst));
    if (nan) atomicOr(&acc->nan, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) cmp_norm_kernel(const T *__restrict__ cand, const T *__restrict__ ref,
                                                            int64_t n, CmpAcc *acc) {
  __shared__ double sn[kThreads / 32], sd[kThreads / 32];
  double num = 0.0, den = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double c = (double)cand[i], r = (double)ref[i];
    const double e = c - r;
    num += e * e;
    den += r * r;
  }
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sn[threadIdx.x >> 5] = num;
    sd[threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) {
      a += sn[w];
      b += sd[w];
    }
    acc->part[2 * blockIdx.x] = a;
    acc->part[2 * blockIdx.x + 1] = b;
  }
}

// one thread sums the CTA partials in CTA order (deterministic)
__global__ void cmp_norm_final_kernel(CmpAcc *acc, int nblocks) {
  double a = 0.0, b = 0.0;
  for (int k = 0; k < nblocks; ++k) {
    a += acc->part[2 * k];
    b += acc->part[2 * k + 1];
  }
  const double rel = sqrt(a) / fmax(sqrt(b), 1e-300);
  acc->worst_bits = (unsigned long long)__double_as_longlong(rel);
}

int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + kThreads * 4 - 1) / (kThreads * 4);
  return (int)(want < (int64_t)sms * kBlocksPerSm ? (want < 1 ? 1 : want) : (int64_t)sms * kBlocksPerSm);
}

}  // namespace

extern "C" size_t b2o_compare_workspace(void) {
  // the accumulator plus room for the norm-wise partials of the largest grid
  return sizeof(CmpAcc) + sizeof(double) * 2 * 256 * kBlocksPerSm;
}

// Asynchronous on `stream`; the verdict is read with b2o_compare_result after
// the stream is synchronised.  host_acc: pinned buffer of
// b2o_compare_workspace() bytes (only the header is copied back).
extern "C" int b2o_compare_device(const void *cand, const void *ref, int64_t n, int elem, int normwise, double tol,
                                  void *ws, void *host_acc, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CmpAcc *acc = (CmpAcc *)ws;
  if (cudaMemsetAsync(acc, 0, sizeof(CmpAcc), s) != cudaSuccess) return -1;
  const int grid = grid_for(n);
  if (normwise) {
    if (elem == B2O_I32) cmp_norm_kernel<int32_t><<<grid, kThreads, 0, s>>>((const int32_t *)cand, (const int32_t *)ref, n, acc);
    else if (elem == B2O_F32) cmp_norm_kernel<float><<<grid, kThreads, 0, s>>>((const float *)cand, (const float *)ref, n, acc);
    else cmp_norm_kernel<double><<<grid, kThreads, 0, s>>>((const double *)cand, (const double *)ref, n, acc);
    cmp_norm_final_kernel<<<1, 1, 0, s>>>(acc, grid);
  } else {
    if (elem == B2O_I32) cmp_elem_kernel<int32_t><<<grid, kThreads, 0, s>>>((const int32_t *)cand, (const int32_t *)ref, n, tol, acc);
    else if (elem == B2O_F32) cmp_elem_kernel<float><<<grid, kThreads, 0, s>>>((const float *)cand, (const float *)ref, n, tol, acc);
    else cmp_elem_kernel<double><<<grid, kThreads, 0, s>>>((const double *)cand, (const double *)ref, n, tol, acc);
  }
  if (cudaGetLastError() != cudaSuccess) return -1;
  return cudaMemcpyAsync(host_acc, acc, sizeof(CmpAcc), cudaMemcpyDeviceToHost, s) == cudaSuccess ? 0 : -1;
}

// after synchronisation: mismatches and worst relative error (+inf when a
// NaN was compared, as on the host); norm-wise: bad = rel > tol
extern "C" void b2o_compare_result(const void *host_acc, int normwise, double tol, uint64_t *bad, double *worst) {
  const CmpAcc *acc = (const CmpAcc *)host_acc;
  union {
    unsigned long long u;
    double d;
  } w;
  w.u = acc->worst_bits;
  if (normwise) {
    *worst = w.d;
    *bad = !(w.d <= tol);
  } else {
    *bad = acc->bad;
    *worst = acc->nan ? INFINITY : w.d;
  }
}

extern "C" void b2o_compare_warm(void) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, (const void *)cmp_elem_kernel<float>);
  cudaFuncGetAttributes(&a, (const void *)cmp_elem_kernel<double>);
  cudaFuncGetAttributes(&a, (const void *)cmp_elem_kernel<int32_t>);
  cudaFuncGetAttributes(&a, (const void *)cmp_norm_kernel<float>);
  cudaFuncGetAttributes(&a, (const void *)cmp_norm_kernel<double>);
  cudaFuncGetAttributes(&a, (const void *)cmp_norm_kernel<int32_t>);
  cudaFuncGetAttributes(&a, cmp_norm_final_kernel);
  cudaGetLastError();
}
