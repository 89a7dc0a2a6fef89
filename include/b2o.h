/*
 * b2o.h — C ABI of the B200 pattern-execution backend (libb2o.so).
 *
 * This is the drop-in boundary for the reference's measurement plugin
 * protocol: the Python evaluator (paper_2011_03602_b200/evaluator.py) that
 * replaces CostModelEvaluator / ExternalCommandEvaluator
 * (reference src/evaluators.py:112-121 and :268-293) calls only these entry
 * points through ctypes.  Plain C types, no exceptions, int status
 * (0 ok, < 0 error, b2o_last_error() for the message).
 *
 * Entry points and the reference interface each one replaces:
 *
 *   b2o_init / b2o_shutdown      one worker thread + stream per B200; replaces
 *                                the serial evaluation loop src/ga.py:270
 *                                (one pattern per GPU)
 *   b2o_app_create ... finalize  the per-pattern build of run_external
 *                                (build_cmd, src/evaluators.py:189-204); here
 *                                the app is compiled once and loaded once
 *   b2o_submit / b2o_wait        ExternalCommandEvaluator.measure
 *                                (src/evaluators.py:288-293) / run_cmd + the
 *                                TIME_SECONDS protocol (src/evaluators.py:206-230)
 *   b2o_result.validity          MeasurementResult.validity vocabulary
 *                                (src/evaluators.py:23-27)
 *   compare inside the runtime   validate_output (src/evaluators.py:129-139)
 *   b2o_gemm_f32 / b2o_fft2d_c64 the DB replacements cublas_gemm / cufft_exec
 *                                (fixtures/sample_db.json:6,15)
 *   b2o_histogram                the DB replacement cuda_histogram
 *                                (fixtures/sample_db.json:20-28)
 */
#ifndef B2O_H
#define B2O_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2O_ABI_VERSION 3

/* validity, identical vocabulary to src/evaluators.py:23-27 */
enum {
  B2O_VALID = 0,
  B2O_NUMERIC_MISMATCH = 1,
  B2O_COMPILE_ERROR = 2,
  B2O_RUNTIME_ERROR = 3,
  B2O_TIMEOUT = 4
};

enum { B2O_DIR_H2D = 0, B2O_DIR_D2H = 1 };
enum { B2O_SIDE_BEFORE = 0, B2O_SIDE_AFTER = 1 };

/* COHERENT: the device-resident variable manager executes the plan at its
 * placements (eliding copies of data that is already valid on the target) and
 * adds counted "unplanned" transfers wherever the plan leaves stale data
 * (SURVEY.md §0.6b-c).  LITERAL: only the plan's copies run; stale reads
 * surface as numeric_mismatch. */
enum { B2O_MODE_COHERENT = 0, B2O_MODE_LITERAL = 1 };

/* one TransferDirective (src/transfers.py:45-53); placement side/anchor */
typedef struct {
  int32_t var_id;
  int32_t dir;          /* B2O_DIR_* */
  int32_t anchor_loop;  /* Placement.anchor_loop: the site is that loop's statement */
  int32_t side;         /* B2O_SIDE_* */
  uint64_t multiplicity;
  int32_t batch_id;
  int32_t reserved;
} b2o_directive;

/* one OffloadPattern (src/patterns.py:51-63) plus its TransferPlan */
typedef struct {
  const uint8_t *gpu_root;   /* n_loops flags: loop id in pattern.gpu_roots */
  int32_t n_loops;
  int32_t n_directives;
  const b2o_directive *directives;
  double priority;           /* larger first (LPT scheduling) */
  double timeout_s;          /* <= 0: no limit */
  int32_t device;            /* worker index, -1 = any */
  int32_t mode;              /* B2O_MODE_* */
  int32_t repeats;           /* timed runs; time_s is the minimum (>= 1) */
  int32_t flags;             /* B2O_FLAG_* */
} b2o_pattern;

/* b2o_pattern.flags: the timed run starts with every array's (pristine)
 * contents already valid in HBM, so the plan's input uploads are elided --
 * the "inputs resident" step of bench.py's value (e2e runs without it). */
#define B2O_FLAG_INPUTS_RESIDENT 2

typedef struct {
  double time_s;             /* wall time of the whole program run (valid only) */
  int32_t validity;
  int32_t worker;
  double max_rel_err;        /* worst |c-r|/|r| over compared outputs */
  uint64_t mismatches;
  uint64_t planned_bytes;    /* bytes moved by plan directives */
  uint64_t elided_bytes;     /* plan bytes skipped because the target was valid */
  uint64_t unplanned_bytes;  /* coherence transfers the plan did not cover */
  uint64_t block_bytes;      /* operand transfers of replaced blocks */
  uint64_t epilogue_bytes;   /* outputs fetched after the run (not timed) */
  uint64_t directive_execs;  /* executed directive instances (== sum multiplicity) */
  uint64_t launches;         /* GPU kernels launched inside the timed region */
  uint64_t stale_reads;      /* LITERAL mode: accesses that saw stale data */
  uint64_t h2d_bytes;        /* all host->device bytes inside the timed run */
  uint64_t d2h_bytes;        /* all device->host bytes inside the timed run */
  char diag[256];
} b2o_result;

int b2o_init(const int32_t *device_ids, int32_t n);
int b2o_shutdown(void);
const char *b2o_last_error(void);
int b2o_num_workers(void);
int b2o_abi_version(void);
/* Broken-worker recovery: after a sticky CUDA error the faulting job returns
 * B2O_RUNTIME_ERROR and the runtime tries to reset that device and rebuild
 * every app replica on it before the next job (b2o_runtime.cu
 * recover_device).  On the B200 driver measured here the reset cannot bring
 * the process's context back (profiles/r02/reset_probe.log), so later jobs
 * on that device return B2O_RUNTIME_ERROR with "device lost" diagnostics;
 * recovery is then a new process -- paper_2011_03602_b200/isolated.py runs
 * the runtime in a child it replaces.  b2o_worker_recoveries counts reset
 * attempts; b2o_debug_inject_fault makes the worker's next job trap on the
 * device (tests only). */
int b2o_debug_inject_fault(int32_t worker);
int64_t b2o_worker_recoveries(int32_t worker);

/* app = one compiled program.  b2o_app_load is SURVEY.md §8(b)'s
 * app_load(model_json, app_spec_json): the IR document (the reference's
 * irdoc.model_to_document, src/irdoc.py:95-166) and the app spec (inputs,
 * outputs, tolerances, block shapes; appspec.py) as JSON text; it runs the
 * package's compiler as a build step (compile_cli.py; B2O_PYTHON picks the
 * interpreter, default python3), sets every variable's initial value and
 * finalises (the all-CPU reference run included).  Status < 0 with the
 * compiler's reason in b2o_last_error for a program it rejects.
 * b2o_app_create is the lower level: a prebuilt host module + cubin. */
int b2o_app_load(const char *model_json, const char *app_spec_json, uint64_t *app);
int b2o_app_num_loops(uint64_t app);                  /* length of b2o_pattern.gpu_root */
int b2o_app_var_id(uint64_t app, const char *name);   /* variable id by name (< 0: none) */
int b2o_app_create(const char *host_module, const char *cubin, uint64_t *app);
int b2o_app_set_initial(uint64_t app, int32_t var_id, const void *data, uint64_t bytes);
int b2o_app_set_reference(uint64_t app, int32_t var_id, const void *data, uint64_t bytes);
int b2o_app_finalize(uint64_t app);          /* per-worker state; reference run if none set */
int b2o_app_get_reference(uint64_t app, int32_t var_id, void *out, uint64_t bytes);
int b2o_app_read(uint64_t app, int32_t worker, int32_t var_id, void *out, uint64_t bytes);
double b2o_app_reference_time(uint64_t app);  /* wall time of the all-CPU reference run */
int b2o_app_destroy(uint64_t app);

int b2o_submit(uint64_t app, const b2o_pattern *patterns, int32_t n, uint64_t *batch);
int b2o_wait(uint64_t batch, b2o_result *results, int32_t n, double timeout_s);

/* device-resident replay (bench): run the pattern once recording every kernel
 * launch, then re-issue that launch sequence `steps` times on the resident
 * data, timed with CUDA events on the worker's stream.  kernel_ms[loop] is the
 * mean device time of one launch of that loop's kernel (0 if never launched). */
int b2o_bench_replay(uint64_t app, int32_t worker, const b2o_pattern *pattern, int32_t warmup, int32_t steps,
                     double *ms_per_step, double *kernel_ms, int32_t n_loops, uint64_t *launches_per_step);

/* hand-written sm_100a kernels behind the block replacements, on device
 * pointers, stream = cudaStream_t (NULL = default) */
int b2o_gemm_f32(const float *A, const float *B, float *C, int64_t m, int64_t n, int64_t k, void *stream);
int b2o_fft2d_c64(const float *x, float *y, int64_t n, void *stream);
int b2o_gemm_impl(void);  /* which GEMM path the build uses: 1 = tcgen05 3xTF32, 0 = SIMT */
/* measurement hook: b2o_gemm_f32 on the tcgen05 path (-2 if the shape does not
 * tile) plus device ms of operand preparation and of the MMA kernel; synchronises */
int b2o_gemm_f32_phases(const float *A, const float *B, float *C, int64_t m, int64_t n, int64_t k, void *stream,
                        double *prep_ms, double *mma_ms);
/* h[d[i]] += 1 for i < n on the device (values outside [0, bins) skipped);
 * elem: element type of h, 0 = int32, 1 = fp32, 2 = fp64 (b2o_module.h b2o_elem) */
int b2o_histogram(const int32_t *d, int64_t n, void *h, int64_t bins, int elem, void *stream);

/* The sequential fp32 sum s = (((s0 + x[0]) + x[1]) + ...) -- every addition
 * rounded to fp32 in index order, the C loop `s = s + x[i]` -- computed in
 * parallel, bit-identical to the loop (binade-segmented integer scan,
 * csrc/b2o_xsum.cu).  x and s_out are device pointers; asynchronous on
 * `stream`.  Used by the opt-in GPU reductions (reductions.py) so an
 * offloaded `gosa = gosa + gs[...]` nest (reference src/screen.py:57-68
 * rejects it) reproduces the CPU loop exactly.  _ws: caller-provided device
 * workspace of b2o_exact_sum_workspace(n) bytes. */
int b2o_exact_sum_f32(const float *x, int64_t n, float s0, float *s_out, void *stream);
size_t b2o_exact_sum_workspace(int64_t n);
int b2o_exact_sum_f32_ws(const float *x, int64_t n, float s0, float *s_out, void *workspace, void *stream);
/* the same in fp64: s = (((s0 + x[0]) + x[1]) + ...) in double, bit-identical
 * to the C loop; the workspace size above covers both formats */
int b2o_exact_sum_f64(const double *x, int64_t n, double s0, double *s_out, void *stream);
int b2o_exact_sum_f64_ws(const double *x, int64_t n, double s0, double *s_out, void *workspace, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* B2O_H */
