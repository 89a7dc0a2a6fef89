// Operations behind opaque library calls (CPU bindings, SURVEY.md Appendix
// A.5) and behind the pattern-DB replacements cublas_gemm / cufft_exec
// (hand-written sm_100a kernels; reference fixtures/sample_db.json:6,15).
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

// host: C = A B, row-major m x k times k x n, double accumulation
void b2o_cpu_gemm(const void *A, const void *B, void *C, int64_t m, int64_t n, int64_t k, int elem);
// host: y = forward 2-D DFT of x (interleaved complex, n x n), double precision
void b2o_cpu_fft2d(const void *x, void *y, int64_t n, int elem);
// host: h[d[i]] += 1 for i < n (values outside [0, bins) skipped), h of b2o_elem elem
void b2o_cpu_histogram(const int32_t *d, int64_t n, void *h, int64_t bins, int elem);

// force-load each file's kernels on the current device (b2o_init)
void b2o_ops_warm(void);
void b2o_gemm_tc_warm(void);
void b2o_gemm_warm(void);
void b2o_xsum_warm(void);
// output comparison on the device (b2o_compare.cu): asynchronous on stream,
// verdict via b2o_compare_result after synchronisation
size_t b2o_compare_workspace(void);
int b2o_compare_device(const void *cand, const void *ref, int64_t n, int elem, int normwise, double tol, void *ws,
                       void *host_acc, void *stream);
void b2o_compare_result(const void *host_acc, int normwise, double tol, uint64_t *bad, double *worst);
void b2o_compare_warm(void);

// forget per-device caches (device allocations, function attributes) after
// the runtime reset that device (broken-worker recovery)
void b2o_ops_forget_device(int dev);
void b2o_gemm_tc_forget_device(int dev);
void b2o_xsum_forget_device(int dev);

#ifdef __cplusplus
}
#endif
