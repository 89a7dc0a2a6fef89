// b2o_runtime.cu — pattern executor, device-resident variable manager and
// worker pool behind include/b2o.h.
//
// One worker thread per B200 owns a CUDA stream and, for every loaded app, a
// full replica of the app state (pinned host working copies, device buffers,
// pristine copies for per-pattern reset).  A job is one candidate pattern:
//
//   reset (untimed) -> run the generated host walk (timed wall clock, all GPU
//   work synchronised) -> fetch outputs -> compare against the reference
//   outputs with the reference's rule (src/evaluators.py:129-139).
//
// The variable manager keeps, per variable, host-valid / device-valid bits.
// Plan directives (src/transfers.py:45-53) execute at their placement hooks
// (the anchor loop's statement, before/after); in COHERENT mode a directive
// whose target copy is already valid is elided, and any access that would
// read stale data triggers a counted "unplanned" transfer.
// Scalars read by a kernel ride in the launch arguments (the H2D of a scalar
// is satisfied by value); scalars written by a kernel land in a device slab.

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/b2o.h"
#include "b2o_module.h"
#include "b2o_ops.h"
#include <nvtx3/nvToolsExt.h>  // header-only: ranges for ncu --nvtx / nsys

namespace {

constexpr size_t kB2oGuard = 256;  // bytes of slack before and after each device array

thread_local std::string g_err;
std::mutex g_mu;

int fail(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return -1;
}

using Clock = std::chrono::steady_clock;

size_t elem_bytes(int elem) { return elem == B2O_F64 ? 8 : 4; }

struct AppShared;

struct Worker {
  int index = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::thread th;
  bool broken = false;        // a sticky CUDA error killed this device's context
  std::string broken_why;
  std::atomic<int> inject_fault{0};  // test hook: trap before the next job's run
  uint64_t recoveries = 0;    // device resets performed after a sticky error
  std::atomic<int64_t> deadline_ns{0};
  std::atomic<b2o_exec *> running{nullptr};
  std::atomic<int> timed_out{0};
};

// Per (app, worker) replica.
struct AppDev {
  AppShared *app = nullptr;
  Worker *w = nullptr;
  CUmodule mod = nullptr;
  std::vector<CUfunction> kfun;
  // dev[v] points kB2oGuard bytes into its allocation (dev_alloc[v]): the
  // vectorised (quad) kernels load whole aligned 16-byte chunks, so a masked
  // lane next to the first/last element may touch up to 12 bytes outside the
  // array; the guard keeps those loads inside the allocation
  std::vector<void *> host, dev, dev_alloc, dev_pristine;
  void *cells = nullptr;     // pinned 8-byte scalar cells
  void *slab = nullptr;      // device scalar slab
  void *slab_init = nullptr; // pinned initial slab contents
  void *scratch = nullptr;   // device scratch for reduction partials (zeroed)
  std::vector<void *> red_bufs;        // exact reductions: per-point terms, per slot
  std::vector<int64_t> red_buf_elems;
  void *xsum_ws = nullptr;             // exact-sum workspace (b2o_exact_sum_workspace)
  size_t xsum_ws_bytes = 0;
  std::vector<void *> dev_ref;         // device copies of the reference outputs (device compare)
  void *cmp_ws = nullptr;              // device compare accumulator (b2o_compare_workspace)
  void *cmp_host = nullptr;            // pinned copy of its header
  std::vector<uint8_t> hv, dv, hmod, dev_dirty, host_touched;
  // lazy restore: host[v] still holds the previous job's values although the
  // state is pristine; the pristine bytes are in the app's pinned copy until
  // a host reader needs host[v] (host_fresh), an upload reads them from the
  // pinned copy, and a full download overwrites host[v] anyway
  std::vector<uint8_t> stale;
  bool lazy_reset = true;
  // chunked asynchronous D2H still arriving in host[v] (progressive reads)
  struct Pending {
    int n = 0, done = 0;
    size_t chunk = 0;
    std::vector<cudaEvent_t> ev;
  };
  std::vector<Pending> pend;
  bool async_d2h = true;
  std::vector<uint8_t> is_root, dev_inside, hook_mask;
  std::vector<std::vector<b2o_directive>> hooks[2];
  b2o_exec ex{};
  int mode = B2O_MODE_COHERENT;
  b2o_result acc{};
  int err_validity = B2O_VALID;
  std::string err;
  bool have_final = false;
  bool recording = false;
  struct Launch {
    int loop;
    std::vector<char> args;
    uint32_t geom[6];
  };
  std::vector<Launch> log;
};

struct AppShared {
  std::string host_path, cubin_path;
  void *dl = nullptr;
  const b2o_module_info *info = nullptr;
  b2o_mod_run_fn run = nullptr;
  std::vector<char> image;
  std::vector<std::vector<char>> initial;    // per var
  std::vector<void *> pinned_initial;        // pinned copy of initial[v] (written arrays; lazy restore)
  std::map<int, std::vector<char>> reference;  // per output var
  bool finalized = false;
  double ref_time = -1.0;
  std::vector<std::unique_ptr<AppDev>> per_worker;
};

struct Job {
  AppShared *app;
  b2o_pattern pat;
  std::vector<uint8_t> roots;
  std::vector<b2o_directive> dirs;
  b2o_result res{};
  struct Batch *batch;
  size_t slot;
};

struct Batch {
  std::vector<Job> jobs;
  size_t remaining = 0;
  std::mutex mu;
  std::condition_variable cv;
};

struct Runtime {
  std::vector<std::unique_ptr<Worker>> workers;
  std::deque<Job *> queue;
  std::mutex qmu;
  std::condition_variable qcv;
  bool stopping = false;
  std::thread watchdog;
  std::map<uint64_t, std::unique_ptr<AppShared>> apps;
  std::map<uint64_t, std::unique_ptr<Batch>> batches;
  uint64_t next_id = 1;
  // broken-worker recovery (under qmu): jobs executing per device, and the
  // devices whose workers must not start new jobs while one is being reset
  std::map<int, int> active;
  std::set<int> paused;
};

Runtime *g_rt = nullptr;

// Driver API through the runtime's entry-point query, so libb2o.so does not
// link libcuda.so.1 and loads (for ABI checks) on machines without a driver.
struct DriverApi {
  decltype(&::cuModuleLoadData) moduleLoadData = nullptr;
  decltype(&::cuModuleGetFunction) moduleGetFunction = nullptr;
  decltype(&::cuModuleUnload) moduleUnload = nullptr;
  decltype(&::cuLaunchKernel) launchKernel = nullptr;
  decltype(&::cuLaunchKernelEx) launchKernelEx = nullptr;
  decltype(&::cuGetErrorString) getErrorString = nullptr;
} drv;

template <typename F>
bool driver_sym(const char *name, F *out) {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
  *out = reinterpret_cast<F>(fn);
  return true;
}

bool load_driver_api() {
  return driver_sym("cuModuleLoadData", &drv.moduleLoadData) &&
         driver_sym("cuModuleGetFunction", &drv.moduleGetFunction) &&
         driver_sym("cuModuleUnload", &drv.moduleUnload) && driver_sym("cuLaunchKernel", &drv.launchKernel) &&
         driver_sym("cuLaunchKernelEx", &drv.launchKernelEx) &&
         driver_sym("cuGetErrorString", &drv.getErrorString);
}

// generated kernels on the worker stream: programmatic stream serialisation
// lets a kernel's launch overlap its predecessor's execution (the kernel's
// b2o_pdl_enter() waits for the predecessor's completion before any access);
// B2O_PDL=0 launches them plainly
CUresult launch_app_kernel(CUfunction f, const uint32_t *geom, CUstream st, void **params) {
  static const bool pdl = !(getenv("B2O_PDL") && atoi(getenv("B2O_PDL")) == 0);
  if (!pdl) return drv.launchKernel(f, geom[0], geom[1], geom[2], geom[3], geom[4], geom[5], 0, st, params, nullptr);
  CUlaunchAttribute at[1];
  at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  at[0].value.programmaticStreamSerializationAllowed = 1;
  CUlaunchConfig cfg = {};
  cfg.gridDimX = geom[0];
  cfg.gridDimY = geom[1];
  cfg.gridDimZ = geom[2];
  cfg.blockDimX = geom[3];
  cfg.blockDimY = geom[4];
  cfg.blockDimZ = geom[5];
  cfg.sharedMemBytes = 0;
  cfg.hStream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return drv.launchKernelEx(&cfg, f, params, nullptr);
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------------------
// variable manager primitives (all on the worker's stream)
// ---------------------------------------------------------------------------

AppDev *D(b2o_exec *ex) { return static_cast<AppDev *>(ex->rt); }

void set_error(AppDev *d, int validity, const std::string &msg) {
  if (d->err_validity == B2O_VALID) {
    d->err_validity = validity;
    d->err = msg;
  }
  d->ex.stop = 1;
}

bool cuda_ok(AppDev *d, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return true;
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorIllegalAddress || e == cudaErrorLaunchFailure || e == cudaErrorIllegalInstruction ||
      e == cudaErrorMisalignedAddress || e == cudaErrorHardwareStackError) {
    d->w->broken = true;
    d->w->broken_why = m;
  }
  set_error(d, B2O_RUNTIME_ERROR, m);
  return false;
}

bool cu_ok(AppDev *d, CUresult r, const char *what) {
  if (r == CUDA_SUCCESS) return true;
  const char *s = nullptr;
  drv.getErrorString(r, &s);
  return cuda_ok(d, cudaErrorUnknown, (std::string(what) + ": " + (s ? s : "?")).c_str());
}

const b2o_var_info &VI(AppDev *d, int v) { return d->app->info->vars[v]; }

size_t var_bytes(AppDev *d, int v) {
  const b2o_var_info &vi = VI(d, v);
  return vi.is_array ? (size_t)vi.length * elem_bytes(vi.elem) : elem_bytes(vi.elem);
}

void par_memcpy(void *dst, const void *src, size_t bytes);

// host[v] made pristine before a host reader or writer uses it (lazy reset)
void host_fresh(AppDev *d, int v) {
  if (!d->stale[v]) return;
  const void *src = d->app->pinned_initial[v] ? d->app->pinned_initial[v] : d->app->initial[v].data();
  par_memcpy(d->host[v], src, d->app->initial[v].size());
  d->stale[v] = 0;
}

void copy_h2d(AppDev *d, int v) {
  // a stale host copy is pristine by definition: upload from the pinned
  // pristine bytes instead of restoring host[v] first
  const void *src = d->stale[v] && d->app->pinned_initial[v] ? d->app->pinned_initial[v] : d->host[v];
  if (d->stale[v] && !d->app->pinned_initial[v]) host_fresh(d, v);
  cuda_ok(d, cudaMemcpyAsync(d->dev[v], src, var_bytes(d, v), cudaMemcpyHostToDevice, d->w->stream),
          "H2D copy");
  d->dev_dirty[v] = 1;
  d->acc.h2d_bytes += var_bytes(d, v);
}

constexpr size_t kAsyncD2hMin = (size_t)4 << 20;   // arrays below this download in one piece
constexpr size_t kAsyncD2hChunk = (size_t)1 << 20;
constexpr int kAsyncD2hMaxChunks = 64;

// block until the first `need` bytes of a pending download are in host[v]
void wait_host(AppDev *d, int v, size_t need) {
  AppDev::Pending &p = d->pend[v];
  while (p.done < p.n && (size_t)p.done * p.chunk < need) {
    cuda_ok(d, cudaEventSynchronize(p.ev[p.done]), "D2H chunk wait");
    ++p.done;
  }
  if (p.done >= p.n) p.n = p.done = 0;
}

void wait_host_all(AppDev *d) {
  for (size_t v = 0; v < d->pend.size(); ++v)
    if (d->pend[v].n) wait_host(d, (int)v, SIZE_MAX);
}

void copy_d2h(AppDev *d, int v, bool async_ok = false) {
  const size_t bytes = var_bytes(d, v);
  if (VI(d, v).is_array && async_ok && d->async_d2h && bytes >= kAsyncD2hMin) {
    // chunked download, one event per chunk: the CPU loop that reads the
    // array starts on the first chunk while the rest is still on the link
    wait_host(d, v, SIZE_MAX);
    AppDev::Pending &p = d->pend[v];
    size_t chunk = std::max(kAsyncD2hChunk, (bytes + kAsyncD2hMaxChunks - 1) / kAsyncD2hMaxChunks);
    chunk = (chunk + 4095) & ~(size_t)4095;
    const int n = (int)((bytes + chunk - 1) / chunk);
    while ((int)p.ev.size() < n) {
      cudaEvent_t e;
      if (!cuda_ok(d, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "D2H event")) return;
      p.ev.push_back(e);
    }
    for (int k = 0; k < n; ++k) {
      const size_t off = (size_t)k * chunk, len = std::min(chunk, bytes - off);
      cuda_ok(d, cudaMemcpyAsync((char *)d->host[v] + off, (const char *)d->dev[v] + off, len,
                                 cudaMemcpyDeviceToHost, d->w->stream),
              "D2H chunk copy");
      cuda_ok(d, cudaEventRecord(p.ev[k], d->w->stream), "D2H chunk event");
    }
    p.n = n;
    p.done = 0;
    p.chunk = chunk;
    d->acc.d2h_bytes += bytes;
    d->host_touched[v] = 1;
    d->stale[v] = 0;  // the whole array is overwritten; readers wait for their chunks
    return;
  }
  if (!VI(d, v).is_array && async_ok && d->async_d2h) {
    // a planned scalar download (e.g. a loop index after a GPU nest) does not
    // stall the host walk: every host reader of the cell waits for its event
    wait_host(d, v, SIZE_MAX);
    AppDev::Pending &p = d->pend[v];
    if (p.ev.empty()) {
      cudaEvent_t e;
      if (!cuda_ok(d, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "D2H event")) return;
      p.ev.push_back(e);
    }
    cuda_ok(d, cudaMemcpyAsync(d->host[v], (char *)d->slab + 8 * v, bytes, cudaMemcpyDeviceToHost, d->w->stream),
            "D2H scalar copy");
    cuda_ok(d, cudaEventRecord(p.ev[0], d->w->stream), "D2H scalar event");
    p.n = 1;
    p.done = 0;
    p.chunk = bytes;
    d->acc.d2h_bytes += bytes;
    d->host_touched[v] = 1;
    return;
  }
  if (VI(d, v).is_array) {
    cuda_ok(d, cudaMemcpyAsync(d->host[v], d->dev[v], var_bytes(d, v), cudaMemcpyDeviceToHost, d->w->stream),
            "D2H copy");
  } else {
    cuda_ok(d, cudaMemcpyAsync(d->host[v], (char *)d->slab + 8 * v, var_bytes(d, v), cudaMemcpyDeviceToHost,
                               d->w->stream),
            "D2H scalar copy");
  }
  cuda_ok(d, cudaStreamSynchronize(d->w->stream), "D2H sync");
  d->acc.d2h_bytes += var_bytes(d, v);
  d->host_touched[v] = 1;
  d->stale[v] = 0;
}

// make the host copy current (coherent mode); async_ok: the caller waits
// for the bytes it reads (progressive CPU loops)
void ensure_host(AppDev *d, int v, bool async_ok = false) {
  if (d->hv[v]) {
    host_fresh(d, v);
    return;
  }
  if (d->mode == B2O_MODE_LITERAL) {
    d->acc.stale_reads++;
    // the program reads its host copy as the plan left it: pristine unless
    // this job changed it -- what an eager reset would have shown
    host_fresh(d, v);
    return;
  }
  copy_d2h(d, v, async_ok);
  d->acc.unplanned_bytes += var_bytes(d, v);
  d->hv[v] = 1;
}

// make the device copy current (arrays)
void ensure_dev(AppDev *d, int v, uint64_t *counter) {
  if (d->dv[v]) return;
  if (d->mode == B2O_MODE_LITERAL && counter == &d->acc.unplanned_bytes) {
    d->acc.stale_reads++;
    return;
  }
  copy_h2d(d, v);
  *counter += var_bytes(d, v);
  d->dv[v] = 1;
}

// an array about to be (fully or partially) overwritten on the device
void prepare_dev_write(AppDev *d, int v, uint64_t *counter) {
  if (d->dv[v]) return;
  if (d->hmod[v]) {
    ensure_dev(d, v, counter);
  } else {
    // never touched by the host since reset: the device buffer already holds
    // the pristine contents (present-by-allocation, no copy needed)
    d->dv[v] = 1;
  }
}

// ---------------------------------------------------------------------------
// callbacks used by generated code
// ---------------------------------------------------------------------------

void host_access_impl(AppDev *d, int32_t set, const b2o_varset *prog) {
  b2o_exec *ex = &d->ex;
  const b2o_varset &all = d->app->info->sets[set];
  const b2o_varset &wr = d->app->info->set_writes[set];
  for (int i = 0; i < all.n && !ex->stop; ++i) {
    const int v = all.vars[i];
    bool progressive = false;
    for (int j = 0; prog && j < prog->n; ++j) progressive |= prog->vars[j] == v;
    if (progressive) {
      ensure_host(d, v, true);
    } else {
      wait_host(d, v, SIZE_MAX);
      ensure_host(d, v);
    }
  }
  for (int i = 0; i < wr.n; ++i) wait_host(d, wr.vars[i], SIZE_MAX);
  for (int i = 0; i < wr.n; ++i) {
    int v = wr.vars[i];
    host_fresh(d, v);
    d->hv[v] = 1;
    d->dv[v] = 0;
    d->hmod[v] = 1;
    d->host_touched[v] = 1;
  }
}

void cb_host_access(b2o_exec *ex, int32_t set) { host_access_impl(D(ex), set, nullptr); }

void cb_host_access_fast(b2o_exec *ex, int32_t set, int32_t progressive) {
  AppDev *d = D(ex);
  host_access_impl(d, set, &d->app->info->sets[progressive]);
}

void cb_host_wait(b2o_exec *ex, int32_t var, int64_t elems) {
  AppDev *d = D(ex);
  if (d->pend[var].n) wait_host(d, var, (size_t)std::max<int64_t>(elems, 0) * elem_bytes(VI(d, var).elem));
}

bool red_reserve(AppDev *d, int32_t slot, int64_t n) {
  if ((int32_t)d->red_bufs.size() <= slot) {
    d->red_bufs.resize(slot + 1, nullptr);
    d->red_buf_elems.resize(slot + 1, 0);
  }
  if (d->red_buf_elems[slot] < n) {
    if (d->red_bufs[slot]) cudaFree(d->red_bufs[slot]);
    d->red_bufs[slot] = nullptr;
    d->red_buf_elems[slot] = 0;
    if (!cuda_ok(d, cudaMalloc(&d->red_bufs[slot], sizeof(double) * (size_t)std::max<int64_t>(n, 1)),
                 "exact reduction buffer"))
      return false;
    d->red_buf_elems[slot] = n;
  }
  const size_t ws = b2o_exact_sum_workspace(n);
  if (d->xsum_ws_bytes < ws) {
    if (d->xsum_ws) cudaFree(d->xsum_ws);
    d->xsum_ws = nullptr;
    d->xsum_ws_bytes = 0;
    if (!cuda_ok(d, cudaMalloc(&d->xsum_ws, ws), "exact-sum workspace")) return false;
    d->xsum_ws_bytes = ws;
  }
  return true;
}

void *cb_red_buf(b2o_exec *ex, int32_t slot, int64_t n) {
  AppDev *d = D(ex);
  return red_reserve(d, slot, n) ? d->red_bufs[slot] : nullptr;
}

void cb_red_exact(b2o_exec *ex, int32_t var, int32_t slot, int64_t n, double s0) {
  AppDev *d = D(ex);
  if (slot >= (int32_t)d->red_bufs.size() || !d->red_bufs[slot]) {
    set_error(d, B2O_RUNTIME_ERROR, "exact reduction without its term buffer");
    return;
  }
  void *cell = (char *)d->slab + 8 * var;
  const int rc = VI(d, var).elem == B2O_F64
                     ? b2o_exact_sum_f64_ws((const double *)d->red_bufs[slot], n, s0, (double *)cell, d->xsum_ws,
                                            d->w->stream)
                     : b2o_exact_sum_f32_ws((const float *)d->red_bufs[slot], n, (float)s0, (float *)cell,
                                            d->xsum_ws, d->w->stream);
  if (rc != 0)
    cuda_ok(d, cudaGetLastError() == cudaSuccess ? cudaErrorUnknown : cudaGetLastError(), "exact in-order sum");
}

void cb_pre_launch(b2o_exec *ex, int32_t loop) {
  AppDev *d = D(ex);
  const b2o_loop_info &li = d->app->info->loops[loop];
  for (int i = 0; i < li.reads.n && !ex->stop; ++i) {
    int v = li.reads.vars[i];
    if (VI(d, v).is_array) {
      ensure_dev(d, v, &d->acc.unplanned_bytes);
    } else {
      wait_host(d, v, SIZE_MAX);  // the launch stub reads the host cell next
      ensure_host(d, v);
    }
  }
  for (int i = 0; i < li.writes.n && !ex->stop; ++i) {
    int v = li.writes.vars[i];
    if (VI(d, v).is_array && d->mode == B2O_MODE_COHERENT) prepare_dev_write(d, v, &d->acc.unplanned_bytes);
  }
}

void cb_launch(b2o_exec *ex, int32_t loop, void *args, uint32_t args_bytes, const uint32_t *geom) {
  AppDev *d = D(ex);
  if (args == nullptr || geom == nullptr) {
    set_error(d, B2O_RUNTIME_ERROR, "loop " + std::to_string(loop) + ": iteration space exceeds 2^32");
    return;
  }
  void *params[] = {args};
  if (d->recording) {
    AppDev::Launch L{loop, std::vector<char>((char *)args, (char *)args + args_bytes), {}};
    std::copy(geom, geom + 6, L.geom);
    d->log.push_back(std::move(L));
  }
  if (!cu_ok(d, launch_app_kernel(d->kfun[loop], geom, (CUstream)d->w->stream, params),
             "cuLaunchKernel"))
    return;
  d->acc.launches++;
  const b2o_loop_info &li = d->app->info->loops[loop];
  for (int i = 0; i < li.writes.n; ++i) {
    int v = li.writes.vars[i];
    d->dv[v] = 1;
    d->hv[v] = 0;
    if (VI(d, v).is_array) d->dev_dirty[v] = 1;
  }
}

void cb_hook(b2o_exec *ex, int32_t loop, int32_t side) {
  AppDev *d = D(ex);
  for (const b2o_directive &dir : d->hooks[side][loop]) {
    if (ex->stop) return;
    int v = dir.var_id;
    d->acc.directive_execs++;
    size_t bytes = var_bytes(d, v);
    bool array = VI(d, v).is_array;
    if (dir.dir == B2O_DIR_H2D) {
      if (!array) continue;  // scalar value rides in the next launch's arguments
      if (d->mode == B2O_MODE_COHERENT && d->dv[v]) {
        d->acc.elided_bytes += bytes;
      } else {
        copy_h2d(d, v);
        d->acc.planned_bytes += bytes;
      }
      d->dv[v] = 1;
    } else {
      if (d->mode == B2O_MODE_COHERENT && d->hv[v]) {
        d->acc.elided_bytes += bytes;
      } else {
        copy_d2h(d, v, true);  // every host reader waits for the bytes it touches
        d->acc.planned_bytes += bytes;
      }
      d->hv[v] = 1;
    }
  }
}

void cb_block(b2o_exec *ex, int32_t block) {
  AppDev *d = D(ex);
  wait_host_all(d);
  const b2o_op_info &op = d->app->info->blocks[block];
  // a library call owns its operand transfers (as cuBLAS/cuFFT on host data)
  int saved = d->mode;
  d->mode = B2O_MODE_COHERENT;
  ensure_dev(d, op.in0, &d->acc.block_bytes);
  if (op.in1 >= 0) ensure_dev(d, op.in1, &d->acc.block_bytes);
  if (op.op == B2O_OP_HISTOGRAM) ensure_dev(d, op.out, &d->acc.block_bytes);  // h += counts
  d->dv[op.out] = 1;  // fully overwritten (gemm, fft) or updated on the device (histogram)
  d->mode = saved;
  if (ex->stop) return;
  int rc = 0;
  if (op.op == B2O_OP_GEMM) {
    if (d->app->info->precision != B2O_F32) {
      set_error(d, B2O_RUNTIME_ERROR, "cublas_gemm replacement supports fp32 apps only");
      return;
    }
    rc = b2o_gemm_f32((const float *)d->dev[op.in0], (const float *)d->dev[op.in1], (float *)d->dev[op.out],
                      op.m, op.n, op.k, d->w->stream);
  } else if (op.op == B2O_OP_HISTOGRAM) {
    rc = b2o_histogram((const int32_t *)d->dev[op.in0], op.n, d->dev[op.out], op.m, VI(d, op.out).elem,
                       d->w->stream);
  } else {
    if (d->app->info->precision != B2O_F32) {
      set_error(d, B2O_RUNTIME_ERROR, "cufft_exec replacement supports fp32 apps only");
      return;
    }
    rc = b2o_fft2d_c64((const float *)d->dev[op.in0], (float *)d->dev[op.out], op.n, d->w->stream);
  }
  if (rc != 0) {
    set_error(d, B2O_RUNTIME_ERROR, std::string("block kernel failed: ") + g_err);
    return;
  }
  cuda_ok(d, cudaGetLastError(), "block launch");
  d->acc.launches++;
  d->dv[op.out] = 1;
  d->hv[op.out] = 0;
  d->dev_dirty[op.out] = 1;
}

void cb_external(b2o_exec *ex, int32_t call) {
  AppDev *d = D(ex);
  wait_host_all(d);
  const b2o_op_info &op = d->app->info->calls[call];
  if (op.op < 0) {
    set_error(d, B2O_RUNTIME_ERROR, "opaque call without a CPU binding");
    return;
  }
  ensure_host(d, op.in0);
  if (op.in1 >= 0) ensure_host(d, op.in1);
  ensure_host(d, op.out);
  if (ex->stop) return;
  int elem = VI(d, op.out).elem;
  if (op.op == B2O_OP_GEMM) {
    b2o_cpu_gemm(d->host[op.in0], d->host[op.in1], d->host[op.out], op.m, op.n, op.k, elem);
  } else if (op.op == B2O_OP_HISTOGRAM) {
    b2o_cpu_histogram((const int32_t *)d->host[op.in0], op.n, d->host[op.out], op.m, elem);
  } else {
    b2o_cpu_fft2d(d->host[op.in0], d->host[op.out], op.n, elem);
  }
  d->hv[op.out] = 1;
  d->dv[op.out] = 0;
  d->hmod[op.out] = 1;
  d->host_touched[op.out] = 1;
}

// ---------------------------------------------------------------------------
// app state
// ---------------------------------------------------------------------------

int load_host_module(AppShared *a) {
  a->dl = dlopen(a->host_path.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!a->dl) return fail("dlopen %s: %s", a->host_path.c_str(), dlerror());
  auto info = (b2o_mod_info_fn)dlsym(a->dl, "b2o_mod_info");
  a->run = (b2o_mod_run_fn)dlsym(a->dl, "b2o_mod_run");
  if (!info || !a->run) return fail("module %s lacks b2o_mod_info/b2o_mod_run", a->host_path.c_str());
  a->info = info();
  if (a->info->abi != B2O_MODULE_ABI) return fail("module ABI %d != runtime ABI %d", a->info->abi, B2O_MODULE_ABI);
  std::ifstream f(a->cubin_path, std::ios::binary);
  if (!f) return fail("cannot read cubin %s", a->cubin_path.c_str());
  a->image.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  a->image.push_back(0);
  a->initial.resize(a->info->n_vars);
  for (int v = 0; v < a->info->n_vars; ++v) {
    const b2o_var_info &vi = a->info->vars[v];
    a->initial[v].assign(vi.is_array ? (size_t)vi.length * elem_bytes(vi.elem) : elem_bytes(vi.elem), 0);
  }
  return 0;
}

// src: an existing replica on another worker whose device arrays already
// hold the initial state -- copied device to device (NVLink peer copy across
// GPUs, a plain copy on the same GPU) instead of one more PCIe upload
int make_replica(AppShared *a, Worker *w, AppDev **out, const AppDev *src = nullptr) {
  auto d = std::make_unique<AppDev>();
  d->app = a;
  d->w = w;
  const b2o_module_info *info = a->info;
  int nv = info->n_vars, nl = info->n_loops;
  if (cudaSetDevice(w->device) != cudaSuccess) return fail("cudaSetDevice(%d)", w->device);
  cudaFree(0);
  CUresult r = drv.moduleLoadData(&d->mod, a->image.data());
  if (r != CUDA_SUCCESS) {
    const char *s = nullptr;
    drv.getErrorString(r, &s);
    return fail("cuModuleLoadData: %s", s ? s : "?");
  }
  d->kfun.assign(nl, nullptr);
  for (int l = 0; l < nl; ++l) {
    if (!info->loops[l].kernel) continue;
    r = drv.moduleGetFunction(&d->kfun[l], d->mod, info->loops[l].kernel);
    if (r != CUDA_SUCCESS) return fail("kernel %s missing from cubin", info->loops[l].kernel);
  }
  d->host.assign(nv, nullptr);
  d->dev.assign(nv, nullptr);
  d->dev_alloc.assign(nv, nullptr);
  d->dev_pristine.assign(nv, nullptr);
  if (cudaHostAlloc(&d->cells, 8 * (size_t)std::max(nv, 1), cudaHostAllocPortable) != cudaSuccess)
    return fail("pinned alloc of scalar cells");
  if (cudaHostAlloc(&d->slab_init, 8 * (size_t)std::max(nv, 1), cudaHostAllocPortable) != cudaSuccess)
    return fail("pinned alloc of slab image");
  memset(d->cells, 0, 8 * (size_t)std::max(nv, 1));
  memset(d->slab_init, 0, 8 * (size_t)std::max(nv, 1));
  if (cudaMalloc(&d->slab, 8 * (size_t)std::max(nv, 1)) != cudaSuccess) return fail("device slab alloc");
  if (cudaMalloc(&d->scratch, B2O_SCRATCH_BYTES) != cudaSuccess) return fail("device scratch alloc");
  cudaMemset(d->scratch, 0, B2O_SCRATCH_BYTES);
  for (int v = 0; v < nv; ++v) {
    const b2o_var_info &vi = info->vars[v];
    size_t bytes = a->initial[v].size();
    if (!vi.is_array) {
      d->host[v] = (char *)d->cells + 8 * v;
      memcpy((char *)d->slab_init + 8 * v, a->initial[v].data(), bytes);
      continue;
    }
    if (cudaHostAlloc(&d->host[v], bytes, cudaHostAllocPortable) != cudaSuccess)
      return fail("pinned alloc %zu B for %s", bytes, vi.name);
    if (cudaMalloc(&d->dev_alloc[v], bytes + 2 * kB2oGuard) != cudaSuccess)
      return fail("device alloc %zu B for %s", bytes, vi.name);
    cudaMemset(d->dev_alloc[v], 0, bytes + 2 * kB2oGuard);
    d->dev[v] = (char *)d->dev_alloc[v] + kB2oGuard;
    memcpy(d->host[v], a->initial[v].data(), bytes);
    if (src != nullptr) {
      if (cudaMemcpyPeer(d->dev[v], w->device, src->dev[v], src->w->device, bytes) != cudaSuccess)
        return fail("initial peer copy of %s", vi.name);
    } else if (cudaMemcpy(d->dev[v], d->host[v], bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      return fail("initial upload of %s", vi.name);  // from the pinned copy
    }
    if (vi.written) {
      if (cudaMalloc(&d->dev_pristine[v], bytes) != cudaSuccess) return fail("pristine alloc for %s", vi.name);
      if (cudaMemcpy(d->dev_pristine[v], d->dev[v], bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
        return fail("pristine copy of %s", vi.name);
    }
  }
  d->hv.assign(nv, 1);
  d->dv.assign(nv, 0);
  d->hmod.assign(nv, 0);
  d->dev_dirty.assign(nv, 0);
  d->host_touched.assign(nv, 0);
  d->stale.assign(nv, 0);
  d->lazy_reset = getenv("B2O_EAGER_RESET") == nullptr;
  if (a->pinned_initial.size() != (size_t)nv) a->pinned_initial.assign(nv, nullptr);
  for (int v = 0; v < nv && d->lazy_reset; ++v) {
    const b2o_var_info &vi = info->vars[v];
    if (!vi.is_array || !vi.written || a->pinned_initial[v]) continue;
    if (cudaHostAlloc(&a->pinned_initial[v], a->initial[v].size(), cudaHostAllocPortable) != cudaSuccess)
      return fail("pinned alloc of the pristine copy of %s", vi.name);
    memcpy(a->pinned_initial[v], a->initial[v].data(), a->initial[v].size());
  }
  d->is_root.assign(std::max(nl, 1), 0);
  d->dev_inside.assign(std::max(nl, 1), 0);
  d->hook_mask.assign(std::max(nl, 1), 0);
  d->hooks[0].assign(nl, {});
  d->hooks[1].assign(nl, {});
  b2o_exec &ex = d->ex;
  ex.rt = d.get();
  ex.host = d->host.data();
  ex.dev = d->dev.data();
  ex.slab = d->slab;
  ex.scratch = d->scratch;
  ex.is_root = d->is_root.data();
  ex.dev_inside = d->dev_inside.data();
  ex.hook_mask = d->hook_mask.data();
  ex.hook = cb_hook;
  ex.host_access = cb_host_access;
  ex.host_access_fast = cb_host_access_fast;
  ex.host_wait = cb_host_wait;
  ex.red_buf = cb_red_buf;
  ex.red_exact = cb_red_exact;
  for (int slot = 0; slot < info->exact_slots && info->exact_elems > 0; ++slot)
    if (!red_reserve(d.get(), slot, info->exact_elems)) return fail("exact reduction buffers");
  if (info->exact_slots > 0) {
    // load the exact-sum kernels now (lazy module loading would otherwise
    // charge the first timed pattern for it)
    if (!red_reserve(d.get(), 0, std::max<int64_t>(info->exact_elems, 1)) ||
        b2o_exact_sum_f32_ws((const float *)d->red_bufs[0], 1, 0.f, (float *)d->slab, d->xsum_ws, w->stream) != 0 ||
        cudaStreamSynchronize(w->stream) != cudaSuccess)
      return fail("exact-sum warm-up");
  }
  d->pend.assign(nv, AppDev::Pending{});
  d->dev_ref.assign(nv, nullptr);
  if (cudaMalloc(&d->cmp_ws, b2o_compare_workspace()) != cudaSuccess) return fail("compare workspace alloc");
  if (cudaHostAlloc(&d->cmp_host, b2o_compare_workspace(), cudaHostAllocPortable) != cudaSuccess)
    return fail("compare result buffer");
  d->async_d2h = getenv("B2O_SYNC_D2H") == nullptr;
  ex.pre_launch = cb_pre_launch;
  ex.launch = cb_launch;
  ex.block = cb_block;
  ex.external = cb_external;
  if (cudaDeviceSynchronize() != cudaSuccess) return fail("replica setup sync");
  *out = d.get();
  a->per_worker[w->index] = std::move(d);
  return 0;
}

// release every resource of one replica (device and pinned host memory,
// the loaded cubin); the caller has selected the device and drained the stream
void free_app_dev(AppShared *a, AppDev *d) {
  for (void *p : d->dev_alloc) if (p) cudaFree(p);
  for (void *p : d->dev_pristine) if (p) cudaFree(p);
  for (size_t v = 0; v < d->host.size(); ++v)
    if (a->info->vars[v].is_array && d->host[v]) cudaFreeHost(d->host[v]);
  if (d->cells) cudaFreeHost(d->cells);
  if (d->slab_init) cudaFreeHost(d->slab_init);
  if (d->slab) cudaFree(d->slab);
  if (d->scratch) cudaFree(d->scratch);
  for (void *p : d->red_bufs) if (p) cudaFree(p);
  if (d->xsum_ws) cudaFree(d->xsum_ws);
  for (void *p : d->dev_ref) if (p) cudaFree(p);
  if (d->cmp_ws) cudaFree(d->cmp_ws);
  if (d->cmp_host) cudaFreeHost(d->cmp_host);
  if (d->mod) drv.moduleUnload(d->mod);
  for (auto &p : d->pend)
    for (cudaEvent_t e : p.ev) cudaEventDestroy(e);
  d->pend.clear();
  d->dev_alloc.clear();
  d->dev_pristine.clear();
  d->host.clear();
  d->red_bufs.clear();
  d->dev_ref.clear();
  d->cmp_ws = nullptr;
  d->cmp_host = nullptr;
  d->cells = nullptr;
  d->slab_init = nullptr;
  d->slab = nullptr;
  d->scratch = nullptr;
  d->xsum_ws = nullptr;
  d->xsum_ws_bytes = 0;
  d->mod = nullptr;
}

void par_memcpy(void *dst, const void *src, size_t bytes) {
  if (bytes < ((size_t)16 << 20)) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t chunk = (bytes + 15) / 16;
#pragma omp parallel for num_threads(16) schedule(static)
  for (int t = 0; t < 16; ++t) {
    size_t off = (size_t)t * chunk;
    if (off < bytes) memcpy((char *)dst + off, (const char *)src + off, std::min(chunk, bytes - off));
  }
}

// restore pristine state; host copies valid, device copies "not present"
void reset_state(AppDev *d) {
  wait_host_all(d);
  const b2o_module_info *info = d->app->info;
  for (int v = 0; v < info->n_vars; ++v) {
    const b2o_var_info &vi = info->vars[v];
    if (!vi.is_array) {
      memcpy(d->host[v], d->app->initial[v].data(), d->app->initial[v].size());
    } else if (vi.written) {
      if (d->host_touched[v]) {
        if (d->lazy_reset)
          d->stale[v] = 1;  // restored on first host use (host_fresh), uploads read the pinned copy
        else
          par_memcpy(d->host[v], d->app->initial[v].data(), d->app->initial[v].size());
      }
      // a device copy a kernel or an upload changed is restored whether or
      // not the host ever saw it: prepare_dev_write treats an array the host
      // did not modify since reset as present-by-allocation (pristine), so a
      // written-but-never-downloaded intermediate must not keep the previous
      // job's values
      if (d->dev_dirty[v])
        cudaMemcpyAsync(d->dev[v], d->dev_pristine[v], d->app->initial[v].size(), cudaMemcpyDeviceToDevice,
                        d->w->stream);
    }
    d->dev_dirty[v] = 0;
    d->host_touched[v] = 0;
  }
  cudaMemcpyAsync(d->slab, d->slab_init, 8 * (size_t)std::max(info->n_vars, 1), cudaMemcpyHostToDevice,
                  d->w->stream);
  cudaStreamSynchronize(d->w->stream);
  std::fill(d->hv.begin(), d->hv.end(), 1);
  std::fill(d->dv.begin(), d->dv.end(), 0);
  std::fill(d->hmod.begin(), d->hmod.end(), 0);
  d->acc = b2o_result{};
  d->err_validity = B2O_VALID;
  d->err.clear();
  d->ex.stop = 0;
}

std::string configure_pattern(AppDev *d, const Job &j) {
  const b2o_module_info *info = d->app->info;
  int nl = info->n_loops;
  if (j.pat.n_loops != nl) return "pattern covers " + std::to_string(j.pat.n_loops) + " loops, program has " +
                                 std::to_string(nl);
  std::fill(d->is_root.begin(), d->is_root.end(), 0);
  std::fill(d->dev_inside.begin(), d->dev_inside.end(), 0);
  std::fill(d->hook_mask.begin(), d->hook_mask.end(), 0);
  for (int l = 0; l < nl; ++l) {
    d->hooks[0][l].clear();
    d->hooks[1][l].clear();
  }
  for (int l = 0; l < nl; ++l) {
    if (info->loops[l].device_op) {
      for (int p = l; p >= 0; p = info->loops[p].parent) d->dev_inside[p] = 1;
    }
    if (!j.roots[l]) continue;
    if (!info->loops[l].kernel)
      return "loop " + std::to_string(l) + " cannot run on the GPU: " +
             (info->loops[l].why_not ? info->loops[l].why_not : "?");
    d->is_root[l] = 1;
    for (int p = info->loops[l].parent; p >= 0; p = info->loops[p].parent) d->dev_inside[p] = 1;
  }
  for (const b2o_directive &dir : j.dirs) {
    if (dir.anchor_loop < 0 || dir.anchor_loop >= nl || dir.var_id < 0 || dir.var_id >= info->n_vars ||
        (dir.side != 0 && dir.side != 1))
      return "malformed transfer directive";
    d->hooks[dir.side][dir.anchor_loop].push_back(dir);
    d->hook_mask[dir.anchor_loop] |= (uint8_t)(1 << dir.side);
  }
  return "";
}

// the reference rule |c - r| <= max(rel * |r|, 1e-12) (src/evaluators.py:129-139)
// per element, typed so the loops vectorise; returns (mismatches, worst rel)
template <typename T>
void compare_elementwise(const T *cand, const T *ref, int64_t n, double tol, uint64_t &bad, double &worst) {
  uint64_t cnt = 0;
  double worst_local = 0.0;
  bool saw_nan = false;
  const int nthr = n > (1 << 18) ? 16 : 1;
#pragma omp parallel for num_threads(nthr) reduction(+ : cnt) reduction(max : worst_local) reduction(|| : saw_nan) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    if (cand[i] == ref[i]) continue;  // the common, bit-exact case: no division
    const double c = (double)cand[i], rr = (double)ref[i];
    const double diff = std::fabs(c - rr);
    const double ar = std::fabs(rr);
    cnt += !(diff <= std::max(tol * ar, 1e-12));
    const double rel = diff / std::max(ar, 1e-30);
    saw_nan = saw_nan || (rel != rel);
    worst_local = rel > worst_local ? rel : worst_local;
  }
  bad = cnt;
  worst = saw_nan ? INFINITY : worst_local;
}

template <typename T>
double normwise_rel(const T *cand, const T *ref, int64_t n) {
  double num = 0.0, den = 0.0;
  const int nthr = n > (1 << 18) ? 16 : 1;
#pragma omp parallel for num_threads(nthr) reduction(+ : num, den) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double c = (double)cand[i], rr = (double)ref[i];
    num += (c - rr) * (c - rr);
    den += rr * rr;
  }
  return std::sqrt(num) / std::max(std::sqrt(den), 1e-300);
}

// coherent runs compare an array output where it is current: on the device
// when its HBM copy is valid (no download of data the program never read on
// the host), else on the host.  LITERAL runs always compare the host copy --
// what the program's host side actually holds (stale reads show there).
bool device_compared(AppDev *d, int v) {
  return d->mode == B2O_MODE_COHERENT && VI(d, v).is_array && d->dv[v] && d->cmp_ws && !getenv("B2O_HOST_COMPARE");
}

void compare_outputs(AppDev *d, b2o_result &r) {
  AppShared *a = d->app;
  const b2o_module_info *info = a->info;
  double worst = 0.0;
  uint64_t bad = 0;
  std::string first_bad;
  for (int o = 0; o < info->n_outputs; ++o) {
    const b2o_output_info &oi = info->outputs[o];
    auto it = a->reference.find(oi.var);
    if (it == a->reference.end()) continue;
    const b2o_var_info &vi = info->vars[oi.var];
    int64_t n = vi.is_array ? vi.length : 1;
    if (!device_compared(d, oi.var)) host_fresh(d, oi.var);
    const void *cand = d->host[oi.var];
    const void *ref = it->second.data();
    uint64_t nbad = 0;
    double w = 0.0;
    if (device_compared(d, oi.var)) {
      // the run left the output current in HBM: compare it there against a
      // device copy of the reference (uploaded once per replica)
      const int normwise = oi.mode == B2O_CMP_NORMWISE;
      if (!d->dev_ref[oi.var]) {
        if (!cuda_ok(d, cudaMalloc(&d->dev_ref[oi.var], it->second.size()), "reference output alloc") ||
            !cuda_ok(d, cudaMemcpy(d->dev_ref[oi.var], ref, it->second.size(), cudaMemcpyHostToDevice),
                     "reference output upload"))
          return;
      }
      if (b2o_compare_device(d->dev[oi.var], d->dev_ref[oi.var], n, vi.elem, normwise, oi.rel_tol, d->cmp_ws,
                             d->cmp_host, d->w->stream) != 0 ||
          !cuda_ok(d, cudaStreamSynchronize(d->w->stream), "device compare")) {
        set_error(d, B2O_RUNTIME_ERROR, "device output comparison failed");
        r.validity = B2O_RUNTIME_ERROR;
        snprintf(r.diag, sizeof r.diag, "%s", d->err.c_str());
        return;
      }
      b2o_compare_result(d->cmp_host, normwise, oi.rel_tol, &nbad, &w);
    } else if (oi.mode == B2O_CMP_NORMWISE) {
      double rel = vi.elem == B2O_I32   ? normwise_rel((const int32_t *)cand, (const int32_t *)ref, n)
                   : vi.elem == B2O_F32 ? normwise_rel((const float *)cand, (const float *)ref, n)
                                        : normwise_rel((const double *)cand, (const double *)ref, n);
      if (!(rel <= oi.rel_tol)) nbad = 1;
      w = rel;
    } else if (vi.elem == B2O_I32) {
      compare_elementwise((const int32_t *)cand, (const int32_t *)ref, n, oi.rel_tol, nbad, w);
    } else if (vi.elem == B2O_F32) {
      compare_elementwise((const float *)cand, (const float *)ref, n, oi.rel_tol, nbad, w);
    } else {
      compare_elementwise((const double *)cand, (const double *)ref, n, oi.rel_tol, nbad, w);
    }
    worst = std::max(worst, w);
    if (nbad && first_bad.empty()) first_bad = vi.name;
    bad += nbad;
  }
  r.max_rel_err = worst;
  r.mismatches = bad;
  if (bad && r.validity == B2O_VALID) {
    r.validity = B2O_NUMERIC_MISMATCH;
    snprintf(r.diag, sizeof r.diag, "output %s differs from the reference (%llu elements, max rel %.3g)",
             first_bad.c_str(), (unsigned long long)bad, worst);
  }
}

// test hook target (b2o_debug_inject_fault): a sticky launch failure
__global__ void b2o_trap_kernel() { asm volatile("trap;"); }

void execute(Worker *w, Job &j) {
  b2o_result &r = j.res;
  r = b2o_result{};
  r.worker = w->index;
  if (w->broken) {
    r.validity = B2O_RUNTIME_ERROR;
    snprintf(r.diag, sizeof r.diag, "device lost: %s", w->broken_why.c_str());
    return;
  }
  AppDev *d = j.app->per_worker[w->index].get();
  if (!d) {
    r.validity = B2O_RUNTIME_ERROR;
    snprintf(r.diag, sizeof r.diag, "app not finalized on worker %d", w->index);
    return;
  }
  cudaSetDevice(w->device);
  std::string why = configure_pattern(d, j);
  if (!why.empty()) {
    r.validity = B2O_COMPILE_ERROR;
    snprintf(r.diag, sizeof r.diag, "%s", why.c_str());
    return;
  }
  d->mode = j.pat.mode == B2O_MODE_LITERAL ? B2O_MODE_LITERAL : B2O_MODE_COHERENT;
  int reps = std::max(1, j.pat.repeats);
  double best = INFINITY;
  b2o_result keep{};
  static const bool trace = getenv("B2O_TRACE") != nullptr;
  auto tr0 = Clock::now();
  double reset_ms = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    auto tr = Clock::now();
    nvtxRangePushA("b2o:reset");
    reset_state(d);
    if (j.pat.flags & B2O_FLAG_INPUTS_RESIDENT)
      for (int v = 0; v < j.app->info->n_vars; ++v)
        if (VI(d, v).is_array) d->dv[v] = 1;  // pristine on both sides after the reset
    nvtxRangePop();
    reset_ms += std::chrono::duration<double, std::milli>(Clock::now() - tr).count();
    w->timed_out = 0;
    w->deadline_ns = j.pat.timeout_s > 0 ? now_ns() + (int64_t)(j.pat.timeout_s * 1e9) : 0;
    w->running = &d->ex;
    if (w->inject_fault.exchange(0)) b2o_trap_kernel<<<1, 1, 0, w->stream>>>();
    auto t0 = Clock::now();
    nvtxRangePushA("b2o:pattern");  // the timed program run
    j.app->run(&d->ex);
    cudaError_t e = cudaStreamSynchronize(w->stream);
    nvtxRangePop();
    wait_host_all(d);  // downloads no CPU loop waited for are complete with the stream
    auto t1 = Clock::now();
    w->running = nullptr;
    w->deadline_ns = 0;
    if (e != cudaSuccess) cuda_ok(d, e, "stream sync");
    double t = std::chrono::duration<double>(t1 - t0).count();
    if (w->timed_out || (j.pat.timeout_s > 0 && t > j.pat.timeout_s))
      set_error(d, B2O_TIMEOUT, "pattern exceeded its timeout");
    if (d->err_validity != B2O_VALID) break;
    if (t < best) {
      best = t;
      keep = d->acc;
    }
  }
  if (d->err_validity != B2O_VALID) {
    r = d->acc;
    r.worker = w->index;
    r.validity = d->err_validity;
    snprintf(r.diag, sizeof r.diag, "%s", d->err.c_str());
    cudaStreamSynchronize(w->stream);
    return;
  }
  r = keep;
  r.worker = w->index;
  r.time_s = best;
  r.validity = B2O_VALID;
  // outputs must be readable on the host for the comparison (untimed)
  const b2o_module_info *info = j.app->info;
  for (int o = 0; o < info->n_outputs; ++o) {
    int v = info->outputs[o].var;
    if (!d->hv[v] && d->mode == B2O_MODE_COHERENT && !device_compared(d, v)) {
      copy_d2h(d, v);
      d->hv[v] = 1;
      r.epilogue_bytes += var_bytes(d, v);
    }
  }
  if (d->err_validity != B2O_VALID) {
    r.validity = d->err_validity;
    snprintf(r.diag, sizeof r.diag, "%s", d->err.c_str());
    return;
  }
  auto tc = Clock::now();
  nvtxRangePushA("b2o:compare");
  compare_outputs(d, r);
  nvtxRangePop();
  d->have_final = true;
  if (trace) {
    auto te = Clock::now();
    fprintf(stderr, "[b2o] job worker=%d reset %.3f ms, run %.3f ms, fetch+compare %.3f ms (compare %.3f), total %.3f ms\n",
            w->index, reset_ms, best * 1e3,
            std::chrono::duration<double, std::milli>(te - tr0).count() - reset_ms - best * 1e3 * reps,
            std::chrono::duration<double, std::milli>(te - tc).count(),
            std::chrono::duration<double, std::milli>(te - tr0).count());
  }
}

// Broken-worker recovery.  A sticky CUDA error (illegal address, trap, ...)
// leaves the device's context unusable: the faulting job came back
// runtime_error, and without recovery every later job on the device would
// too.  The first broken worker of the device pauses the device (no new job
// starts on it), waits for the jobs still running there to finish (they fail
// fast on the dead context), resets the device, recreates the workers'
// streams and every app's replica on it from the host copy of the initial
// state, and resumes the queue.  Jobs running on a sibling worker of the same
// device at the moment of the fault return runtime_error; queued jobs run
// after the reset.  cudaDeviceReset destroys the primary context, so device
// memory another library allocated in this process on that device (e.g.
// torch tensors) is lost too.
void recover_device(Worker *w) {
  const int dev = w->device;
  {
    std::unique_lock<std::mutex> lk(g_rt->qmu);
    if (!w->broken) return;
    if (g_rt->paused.count(dev)) {  // a sibling worker is resetting the device
      g_rt->qcv.wait(lk, [&] { return g_rt->stopping || !g_rt->paused.count(dev); });
      return;
    }
    g_rt->paused.insert(dev);
    g_rt->qcv.wait(lk, [&] { return g_rt->active[dev] == 0; });
  }
  std::string why;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaSetDevice(dev);
    cudaError_t e = cudaDeviceReset();
    if (e != cudaSuccess) why = std::string("cudaDeviceReset: ") + cudaGetErrorString(e);
    cudaSetDevice(dev);
    e = cudaFree(0);
    if (e != cudaSuccess && why.empty()) why = std::string("context re-creation: ") + cudaGetErrorString(e);
    cudaGetLastError();
    b2o_ops_forget_device(dev);
    b2o_gemm_tc_forget_device(dev);
    b2o_xsum_forget_device(dev);
    std::vector<Worker *> mine;
    for (auto &x : g_rt->workers)
      if (x->device == dev) mine.push_back(x.get());
    for (Worker *x : mine) {
      x->stream = nullptr;  // destroyed with the context
      e = cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking);
      if (e != cudaSuccess && why.empty()) why = std::string("stream re-creation: ") + cudaGetErrorString(e);
    }
    b2o_ops_warm();
    b2o_gemm_tc_warm();
    b2o_gemm_warm();
    b2o_xsum_warm();
    b2o_compare_warm();
    for (auto &kv : g_rt->apps) {
      AppShared *a = kv.second.get();
      if (!a->finalized) continue;
      for (Worker *x : mine) {
        // the replica's device memory, pinned buffers, events and module went
        // with the context: drop the bookkeeping only
        delete a->per_worker[x->index].release();
        AppDev *d = nullptr;
        if (why.empty() && make_replica(a, x, &d, nullptr) != 0) why = "replica rebuild: " + g_err;
      }
    }
    for (Worker *x : mine) {
      ++x->recoveries;
      if (why.empty()) {
        x->broken = false;
        x->broken_why.clear();
      } else {
        x->broken = true;
        x->broken_why = "device reset after a sticky error failed: " + why;
      }
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_rt->qmu);
    g_rt->paused.erase(dev);
  }
  g_rt->qcv.notify_all();
}

void worker_loop(Worker *w) {
  cudaSetDevice(w->device);
  for (;;) {
    Job *j = nullptr;
    {
      std::unique_lock<std::mutex> lk(g_rt->qmu);
      g_rt->qcv.wait(lk, [&] {
        if (g_rt->stopping) return true;
        if (g_rt->paused.count(w->device)) return false;  // the device is being reset
        for (Job *q : g_rt->queue)
          if (q->pat.device < 0 || q->pat.device == w->index) return true;
        return false;
      });
      if (g_rt->stopping) return;
      for (auto it = g_rt->queue.begin(); it != g_rt->queue.end(); ++it) {
        if ((*it)->pat.device < 0 || (*it)->pat.device == w->index) {
          j = *it;
          g_rt->queue.erase(it);
          ++g_rt->active[w->device];
          break;
        }
      }
    }
    if (!j) continue;
    execute(w, *j);
    {
      std::lock_guard<std::mutex> q(g_rt->qmu);
      --g_rt->active[w->device];
    }
    g_rt->qcv.notify_all();
    {
      Batch *b = j->batch;
      std::lock_guard<std::mutex> lk(b->mu);
      if (--b->remaining == 0) b->cv.notify_all();
    }
    if (w->broken) recover_device(w);
  }
}

void watchdog_loop() {
  while (true) {
    {
      std::lock_guard<std::mutex> lk(g_rt->qmu);
      if (g_rt->stopping) return;
    }
    int64_t t = now_ns();
    for (auto &w : g_rt->workers) {
      int64_t dl = w->deadline_ns.load();
      b2o_exec *ex = w->running.load();
      if (dl > 0 && ex && t > dl) {
        w->timed_out = 1;
        ex->stop = 1;
      }
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
}

AppShared *find_app(uint64_t id) {
  if (!g_rt) return nullptr;
  auto it = g_rt->apps.find(id);
  return it == g_rt->apps.end() ? nullptr : it->second.get();
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

const char *b2o_last_error(void) { return g_err.c_str(); }
int b2o_abi_version(void) { return B2O_ABI_VERSION; }

int b2o_init(const int32_t *device_ids, int32_t n) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_rt) return fail("b2o already initialised");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return fail("no CUDA device visible");
  cudaFree(0);
  if (!load_driver_api()) return fail("CUDA driver entry points unavailable");
  g_rt = new Runtime();
  std::vector<int> ids;
  if (n <= 0 || !device_ids) {
    for (int i = 0; i < count; ++i) ids.push_back(i);
  } else {
    ids.assign(device_ids, device_ids + n);
  }
  for (size_t i = 0; i < ids.size(); ++i) {
    if (ids[i] < 0 || ids[i] >= count) {
      delete g_rt;
      g_rt = nullptr;
      return fail("device %d out of range (%d visible)", ids[i], count);
    }
    auto w = std::make_unique<Worker>();
    w->index = (int)i;
    w->device = ids[i];
    cudaSetDevice(w->device);
    if (cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete g_rt;
      g_rt = nullptr;
      return fail("stream creation on device %d", ids[i]);
    }
    b2o_ops_warm();
    b2o_gemm_tc_warm();
    b2o_gemm_warm();
    b2o_xsum_warm();
    b2o_compare_warm();
    g_rt->workers.push_back(std::move(w));
  }
  for (auto &w : g_rt->workers) w->th = std::thread(worker_loop, w.get());
  g_rt->watchdog = std::thread(watchdog_loop);
  return 0;
}

int b2o_num_workers(void) { return g_rt ? (int)g_rt->workers.size() : 0; }

int b2o_debug_inject_fault(int32_t worker) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_rt || worker < 0 || worker >= (int)g_rt->workers.size()) return fail("bad worker %d", worker);
  g_rt->workers[worker]->inject_fault = 1;
  return 0;
}

int64_t b2o_worker_recoveries(int32_t worker) {
  if (!g_rt || worker < 0 || worker >= (int)g_rt->workers.size()) return -1;
  return (int64_t)g_rt->workers[worker]->recoveries;
}

int b2o_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_rt) return 0;
  {
    std::lock_guard<std::mutex> q(g_rt->qmu);
    g_rt->stopping = true;
  }
  g_rt->qcv.notify_all();
  for (auto &w : g_rt->workers) w->th.join();
  g_rt->watchdog.join();
  for (auto &kv : g_rt->apps) {
    AppShared *a = kv.second.get();
    for (auto &d : a->per_worker) {
      if (!d) continue;
      free_app_dev(a, d.get());
    }
    for (void *p : a->pinned_initial)
      if (p) cudaFreeHost(p);
    a->pinned_initial.clear();
  }
  for (auto &w : g_rt->workers) {
    cudaSetDevice(w->device);
    cudaStreamDestroy(w->stream);
  }
  delete g_rt;
  g_rt = nullptr;
  return 0;
}

int b2o_app_create(const char *host_module, const char *cubin, uint64_t *app) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_rt) return fail("b2o_init not called");
  auto a = std::make_unique<AppShared>();
  a->host_path = host_module;
  a->cubin_path = cubin;
  if (load_host_module(a.get()) != 0) return -1;
  a->per_worker.resize(g_rt->workers.size());
  uint64_t id = g_rt->next_id++;
  g_rt->apps[id] = std::move(a);
  *app = id;
  return 0;
}

// b2o_app_load: the compile service (paper_2011_03602_b200/compile_cli.py)
// run as a build step, then create + initial state + finalize.
namespace {
std::string repo_root() {
  Dl_info info;
  if (!dladdr((void *)&b2o_app_load, &info) || !info.dli_fname) return ".";
  std::string p = info.dli_fname;  // <root>/paper_2011_03602_b200/libb2o.so
  for (int up = 0; up < 2; ++up) {
    size_t k = p.find_last_of('/');
    p = k == std::string::npos ? "." : p.substr(0, k);
  }
  return p.empty() ? "/" : p;
}

bool write_file(const std::string &path, const char *text) {
  FILE *f = fopen(path.c_str(), "wb");
  if (!f) return false;
  size_t n = strlen(text);
  bool ok = fwrite(text, 1, n, f) == n;
  return fclose(f) == 0 && ok;
}

std::string shell_quote(const std::string &s) {
  std::string o = "'";
  for (char c : s) o += c == '\'' ? std::string("'\\''") : std::string(1, c);
  return o + "'";
}
}  // namespace

int b2o_app_load(const char *model_json, const char *app_spec_json, uint64_t *app) {
  if (!model_json || !app_spec_json || !app) return fail("b2o_app_load: null argument");
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_rt) return fail("b2o_init not called");
  }
  char dir[] = "/tmp/b2o_load_XXXXXX";
  if (!mkdtemp(dir)) return fail("b2o_app_load: mkdtemp failed");
  const std::string d = dir;
  auto cleanup = [&] { std::system(("rm -rf " + shell_quote(d)).c_str()); };
  if (!write_file(d + "/doc.json", model_json) || !write_file(d + "/spec.json", app_spec_json)) {
    cleanup();
    return fail("b2o_app_load: cannot write the request");
  }
  const char *py = getenv("B2O_PYTHON");
  const std::string root = repo_root();
  const std::string cmd = "cd " + shell_quote(root) + " && PYTHONPATH=" + shell_quote(root) +
                          "${PYTHONPATH:+:$PYTHONPATH} " + shell_quote(py && *py ? py : "python3") +
                          " -m paper_2011_03602_b200.compile_cli " + shell_quote(d + "/doc.json") + " " +
                          shell_quote(d + "/spec.json") + " " + shell_quote(d) + " 2> " +
                          shell_quote(d + "/err.txt") + " > /dev/null";
  const int rc = std::system(cmd.c_str());
  if (rc != 0) {
    std::string why;
    if (FILE *f = fopen((d + "/err.txt").c_str(), "rb")) {
      char buf[512];
      size_t n = fread(buf, 1, sizeof buf - 1, f);
      buf[n] = 0;
      fclose(f);
      why = buf;
    }
    cleanup();
    return fail("b2o_app_load: compile service failed (%d): %s", rc, why.c_str());
  }
  std::ifstream man(d + "/manifest.txt");
  std::string kind, host, cubin;
  struct Init {
    int id;
    uint64_t bytes;
    std::string path;
  };
  std::vector<Init> inits;
  while (man >> kind) {
    if (kind == "host") man >> host;
    else if (kind == "cubin") man >> cubin;
    else if (kind == "loops") { int n; man >> n; }
    else if (kind == "var") {
      Init v;
      std::string name;
      man >> v.id >> v.bytes >> v.path >> name;
      inits.push_back(v);
    } else {
      std::string rest;
      std::getline(man, rest);
    }
  }
  if (host.empty() || cubin.empty()) {
    cleanup();
    return fail("b2o_app_load: malformed manifest");
  }
  uint64_t id = 0;
  if (b2o_app_create(host.c_str(), cubin.c_str(), &id) != 0) {
    cleanup();
    return -1;
  }
  for (const Init &v : inits) {
    std::vector<char> buf(v.bytes);
    FILE *f = fopen(v.path.c_str(), "rb");
    bool ok = f && fread(buf.data(), 1, v.bytes, f) == v.bytes;
    if (f) fclose(f);
    if (!ok || b2o_app_set_initial(id, v.id, buf.data(), v.bytes) != 0) {
      cleanup();
      b2o_app_destroy(id);
      return ok ? -1 : fail("b2o_app_load: cannot read the initial value of var %d", v.id);
    }
  }
  cleanup();
  if (b2o_app_finalize(id) != 0) {
    std::string why = g_err;
    b2o_app_destroy(id);
    return fail("%s", why.c_str());
  }
  *app = id;
  return 0;
}

int b2o_app_num_loops(uint64_t app) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  return a ? a->info->n_loops : fail("unknown app");
}

int b2o_app_var_id(uint64_t app, const char *name) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a || !name) return fail("unknown app");
  for (int v = 0; v < a->info->n_vars; ++v)
    if (strcmp(a->info->vars[v].name, name) == 0) return v;
  return fail("no variable named %s", name);
}

int b2o_app_set_initial(uint64_t app, int32_t var_id, const void *data, uint64_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app %llu", (unsigned long long)app);
  if (a->finalized) return fail("app already finalized");
  if (var_id < 0 || var_id >= a->info->n_vars) return fail("bad var id %d", var_id);
  if (bytes != a->initial[var_id].size())
    return fail("var %s: %llu bytes given, %zu expected", a->info->vars[var_id].name, (unsigned long long)bytes,
                a->initial[var_id].size());
  memcpy(a->initial[var_id].data(), data, bytes);
  return 0;
}

int b2o_app_set_reference(uint64_t app, int32_t var_id, const void *data, uint64_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app");
  if (var_id < 0 || var_id >= a->info->n_vars) return fail("bad var id %d", var_id);
  if (bytes != a->initial[var_id].size()) return fail("reference size mismatch for %s", a->info->vars[var_id].name);
  a->reference[var_id].assign((const char *)data, (const char *)data + bytes);
  return 0;
}

int b2o_app_finalize(uint64_t app) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app");
  if (a->finalized) return 0;
  for (auto &w : g_rt->workers) {
    AppDev *d = nullptr;
    // worker 0 uploads over PCIe, the others copy from it over NVLink
    const AppDev *src = w->index > 0 ? a->per_worker[0].get() : nullptr;
    if (make_replica(a, w.get(), &d, src) != 0) return -1;
  }
  a->finalized = true;
  bool need_ref = false;
  for (int o = 0; o < a->info->n_outputs; ++o)
    if (!a->reference.count(a->info->outputs[o].var)) need_ref = true;
  if (need_ref) {
    // the original program: every loop on the CPU (genome 0...0)
    Worker *w = g_rt->workers[0].get();
    AppDev *d = a->per_worker[0].get();
    Job j{};
    j.app = a;
    j.pat.n_loops = a->info->n_loops;
    j.pat.repeats = 1;
    j.pat.device = 0;
    j.roots.assign(a->info->n_loops, 0);
    // run on the caller thread with the worker's stream: the worker is idle
    // because no batch can reference this app before finalize returns
    execute(w, j);
    if (j.res.validity != B2O_VALID && j.res.validity != B2O_NUMERIC_MISMATCH)
      return fail("reference run failed: %s", j.res.diag);
    a->ref_time = j.res.time_s;
    for (int o = 0; o < a->info->n_outputs; ++o) {
      int v = a->info->outputs[o].var;
      if (a->reference.count(v)) continue;
      a->reference[v].assign((const char *)d->host[v], (const char *)d->host[v] + a->initial[v].size());
    }
  }
  // device copies of the reference outputs for the on-device comparison,
  // uploaded now so no measurement call pays for them
  for (auto &dp : a->per_worker) {
    cudaSetDevice(dp->w->device);
    for (int o = 0; o < a->info->n_outputs; ++o) {
      int v = a->info->outputs[o].var;
      auto it = a->reference.find(v);
      if (!a->info->vars[v].is_array || it == a->reference.end() || dp->dev_ref[v]) continue;
      if (cudaMalloc(&dp->dev_ref[v], it->second.size()) != cudaSuccess ||
          cudaMemcpy(dp->dev_ref[v], it->second.data(), it->second.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail("reference output upload for %s", a->info->vars[v].name);
    }
  }
  return 0;
}

double b2o_app_reference_time(uint64_t app) {
  AppShared *a = find_app(app);
  return a ? a->ref_time : -1.0;
}

int b2o_app_get_reference(uint64_t app, int32_t var_id, void *out, uint64_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app");
  auto it = a->reference.find(var_id);
  if (it == a->reference.end()) return fail("no reference for var %d", var_id);
  if (bytes != it->second.size()) return fail("reference size mismatch");
  memcpy(out, it->second.data(), bytes);
  return 0;
}

int b2o_app_read(uint64_t app, int32_t worker, int32_t var_id, void *out, uint64_t bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a || worker < 0 || worker >= (int)a->per_worker.size() || !a->per_worker[worker])
    return fail("unknown app/worker");
  AppDev *d = a->per_worker[worker].get();
  if (var_id < 0 || var_id >= a->info->n_vars) return fail("bad var id");
  if (bytes != a->initial[var_id].size()) return fail("size mismatch");
  if (!d->hv[var_id]) {
    // compared on the device and never downloaded: read the HBM copy
    cudaSetDevice(d->w->device);
    const void *src = a->info->vars[var_id].is_array ? d->dev[var_id] : (const char *)d->slab + 8 * var_id;
    if (cudaMemcpy(out, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return fail("device read of var %d", var_id);
    return 0;
  }
  if (d->stale[var_id]) {  // untouched since the lazy reset: the pristine bytes
    const void *src = a->pinned_initial[var_id] ? a->pinned_initial[var_id] : a->initial[var_id].data();
    memcpy(out, src, bytes);
    return 0;
  }
  memcpy(out, d->host[var_id], bytes);
  return 0;
}

int b2o_app_destroy(uint64_t app) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app");
  for (auto &d : a->per_worker) {
    if (!d) continue;
    cudaSetDevice(d->w->device);
    cudaStreamSynchronize(d->w->stream);
    free_app_dev(a, d.get());
  }
  for (void *p : a->pinned_initial)
    if (p) cudaFreeHost(p);
  a->pinned_initial.clear();
  if (a->dl) dlclose(a->dl);
  g_rt->apps.erase(app);
  return 0;
}

int b2o_bench_replay(uint64_t app, int32_t worker, const b2o_pattern *pattern, int32_t warmup, int32_t steps,
                     double *ms_per_step, double *kernel_ms, int32_t n_loops, uint64_t *launches_per_step) {
  std::lock_guard<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a || !a->finalized) return fail("unknown or unfinalized app");
  if (worker < 0 || worker >= (int)a->per_worker.size()) return fail("bad worker");
  AppDev *d = a->per_worker[worker].get();
  Worker *w = d->w;
  if (n_loops != a->info->n_loops) return fail("kernel_ms has %d slots, program has %d loops", n_loops,
                                               a->info->n_loops);
  cudaSetDevice(w->device);
  Job j{};
  j.app = a;
  j.pat = *pattern;
  j.roots.assign(pattern->gpu_root, pattern->gpu_root + pattern->n_loops);
  j.dirs.assign(pattern->directives, pattern->directives + pattern->n_directives);
  std::string why = configure_pattern(d, j);
  if (!why.empty()) return fail("%s", why.c_str());
  d->mode = B2O_MODE_COHERENT;
  reset_state(d);
  d->log.clear();
  d->recording = true;
  a->run(&d->ex);
  d->recording = false;
  if (cudaStreamSynchronize(w->stream) == cudaSuccess) wait_host_all(d);
  if (cudaStreamSynchronize(w->stream) != cudaSuccess || d->err_validity != B2O_VALID)
    return fail("recording run failed: %s", d->err.c_str());
  if (d->log.empty()) return fail("pattern launches no kernel");
  auto replay = [&]() -> bool {
    for (auto &L : d->log) {
      void *params[] = {L.args.data()};
      if (launch_app_kernel(d->kfun[L.loop], L.geom, (CUstream)w->stream, params) != CUDA_SUCCESS)
        return false;
    }
    return true;
  };
  for (int i = 0; i < warmup; ++i)
    if (!replay()) return fail("replay launch failed");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, w->stream);
  for (int i = 0; i < steps; ++i)
    if (!replay()) return fail("replay launch failed");
  cudaEventRecord(e1, w->stream);
  if (cudaEventSynchronize(e1) != cudaSuccess) return fail("replay failed: %s", cudaGetErrorString(cudaGetLastError()));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_per_step = steps > 0 ? ms / steps : 0.0;
  *launches_per_step = d->log.size();
  // per-kernel device time: that loop's recorded launches back to back,
  // one event pair around `passes` repetitions
  std::vector<double> sum(n_loops, 0.0);
  std::vector<int> cnt(n_loops, 0);
  int passes = std::max(3, std::min(steps, 20));
  for (int l = 0; l < n_loops; ++l) {
    std::vector<const AppDev::Launch *> mine;
    for (auto &L : d->log)
      if (L.loop == l) mine.push_back(&L);
    if (mine.empty()) continue;
    auto issue = [&]() {
      for (const AppDev::Launch *L : mine) {
        void *params[] = {(void *)L->args.data()};
        launch_app_kernel(d->kfun[l], L->geom, (CUstream)w->stream, params);
      }
    };
    issue();
    cudaEventRecord(e0, w->stream);
    for (int pss = 0; pss < passes; ++pss) issue();
    cudaEventRecord(e1, w->stream);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    sum[l] = t;
    cnt[l] = passes * (int)mine.size();
  }
  for (int l = 0; l < n_loops; ++l) kernel_ms[l] = cnt[l] ? sum[l] / cnt[l] : 0.0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  d->log.clear();
  return 0;
}

int b2o_submit(uint64_t app, const b2o_pattern *patterns, int32_t n, uint64_t *batch) {
  std::unique_lock<std::mutex> lk(g_mu);
  AppShared *a = find_app(app);
  if (!a) return fail("unknown app");
  if (!a->finalized) return fail("app not finalized");
  auto b = std::make_unique<Batch>();
  b->jobs.resize(n);
  b->remaining = n;
  for (int i = 0; i < n; ++i) {
    Job &j = b->jobs[i];
    j.app = a;
    j.pat = patterns[i];
    j.roots.assign(patterns[i].gpu_root, patterns[i].gpu_root + std::max(patterns[i].n_loops, 0));
    j.dirs.assign(patterns[i].directives, patterns[i].directives + std::max(patterns[i].n_directives, 0));
    j.batch = b.get();
    j.slot = i;
    if (j.pat.device >= (int)g_rt->workers.size()) return fail("pattern %d targets worker %d", i, j.pat.device);
  }
  uint64_t id = g_rt->next_id++;
  Batch *raw = b.get();
  g_rt->batches[id] = std::move(b);
  lk.unlock();
  {
    std::lock_guard<std::mutex> q(g_rt->qmu);
    std::vector<Job *> order;
    for (auto &j : raw->jobs) order.push_back(&j);
    std::stable_sort(order.begin(), order.end(),
                     [](const Job *x, const Job *y) { return x->pat.priority > y->pat.priority; });
    for (Job *j : order) g_rt->queue.push_back(j);
  }
  g_rt->qcv.notify_all();
  *batch = id;
  return 0;
}

int b2o_wait(uint64_t batch, b2o_result *results, int32_t n, double timeout_s) {
  Batch *b = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_rt) return fail("not initialised");
    auto it = g_rt->batches.find(batch);
    if (it == g_rt->batches.end()) return fail("unknown batch");
    b = it->second.get();
  }
  {
    std::unique_lock<std::mutex> lk(b->mu);
    if (timeout_s > 0) {
      if (!b->cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return b->remaining == 0; }))
        return fail("batch wait timed out");
    } else {
      b->cv.wait(lk, [&] { return b->remaining == 0; });
    }
  }
  if (n != (int)b->jobs.size()) return fail("batch has %zu results, %d requested", b->jobs.size(), n);
  for (int i = 0; i < n; ++i) results[i] = b->jobs[i].res;
  std::lock_guard<std::mutex> lk(g_mu);
  g_rt->batches.erase(batch);
  return 0;
}

}  // extern "C"
