// b2o_xsum.cu — the sequential fp32 sum  s = s + x[0] + x[1] + ... (each
// addition rounded to fp32, in index order: the C loop `gosa = gosa + gs[i]`)
// computed in parallel on the GPU, bit-identical to the sequential loop.
//
// Why it parallelises: while the running sum s stays inside one binade
// [2^e, 2^(e+1)) it is an integer S in units u = 2^(e-23), S in [2^23, 2^24),
// and (unless x is exactly half-way between two multiples of u)
//
//     fl(s + x) = (S + r) u,   r = round-to-nearest(x / u),
//
// provided the exact sum stays inside the binade.  r depends on x and e only,
// not on s, so for a fixed binade the effect of a whole run of elements is an
// integer sum -- associative, hence scan-able -- plus the range of the
// running integer prefix (to check that s never left the binade).  Every
// element's validity condition is kept conservative:
//
//     S + P_j + r_j - 1 >= 2^23   and   S + P_j + r_j + 1 <= 2^24
//
// (P_j = r_0 + ... + r_(j-1)); a half-way x (a tie: the result would depend
// on the parity of S), an infinity / NaN, or an x too large for the binade
// flags the run as unusable.
//
// Three kernels on the caller's stream:
//   A  bound:    B = |s0| + sum |x| (double)  -> the binade window: the 16
//                binades below B's (any |s_j| <= B up to rounding slack);
//   B  summarise: per chunk of 256 elements (one warp) and per window binade:
//                (P, min prefix - 1, max prefix + 1, flags); a CTA of 32 warps
//                also merges its 32 chunks into a super-chunk summary;
//   C  compose:  one warp walks the super-chunks in order; a super-chunk (or
//                chunk) whose summary is valid for the current (S, e) is
//                applied in O(1); otherwise it descends into chunks, and a
//                chunk that is not valid either (a binade crossing, a tie, an
//                s <= 0 or outside the window) is added element by element
//                with __fadd_rn -- the definition itself.
// Summaries of the next super-chunk / chunk are prefetched (lane k holds the
// binade-k record) so the serial walk does not wait on memory.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <map>

#include "../../include/b2o.h"

namespace {

constexpr int XS_CHUNK = 256;        // elements per chunk (one warp, 8 per lane)
constexpr int XS_PER_LANE = XS_CHUNK / 32;
constexpr int XS_SUPER = 32;         // chunks per super-chunk (one CTA of 32 warps)
constexpr int XS_W = 16;             // binades in the window

// A run's effect for one binade, in units u.  Valid summaries have |P|, |lo|,
// |hi| <= 2^24 + 1 (the running integer stays in [2^23, 2^24)); anything
// larger is flagged, which also keeps every int32 sum below overflow.
struct Summ {
  int P;      // sum of r
  int lo;     // min over j of (P_(j+1) - 1)
  int hi;     // max over j of (P_(j+1) + 1)
  int flags;  // nonzero: unusable for this binade
};

constexpr int kLoEmpty = 0x7FFFFFFF, kHiEmpty = -0x7FFFFFFF - 1;
constexpr int kBig = 1 << 25;

// r = round(x / 2^(e-23)) with the tie / range flag; x as raw bits.
// Branch-free (the 16 lanes of a half-warp evaluate 16 different binades).
// |x| >= 2^(e+1) (d > 0) can never keep the sum inside the binade: flagged.
__device__ __forceinline__ int units(uint32_t bits, int e, int &flag) {
  const uint32_t exr = (bits >> 23) & 0xFFu;
  const uint32_t m = (bits & 0x7FFFFFu) | (exr ? 0x800000u : 0u);
  const int ex = exr ? (int)exr - 127 : -126;
  const int d = ex - e;
  const int sh = min(max(-d, 1), 31);
  const uint32_t q = m >> sh, rem = m & ((1u << sh) - 1u), half = 1u << (sh - 1);
  const int dn = (int)q + (rem > half ? 1 : 0);
  // round half to even would be decided by S's parity: flag the tie
  flag |= (exr == 0xFFu) | (d > 0) | (d < 0 && rem == half);
  const int r = d == 0 ? (int)m : (d < 0 ? dn : 0);
  return (bits >> 31) ? -r : r;
}

__device__ __forceinline__ bool big(const Summ &a) {
  return a.P > kBig || a.P < -kBig || (a.lo != kLoEmpty && (a.lo > kBig || a.lo < -kBig)) ||
         (a.hi != kHiEmpty && (a.hi > kBig || a.hi < -kBig));
}

// a then b
__device__ __forceinline__ Summ merge(const Summ &a, const Summ &b) {
  if (b.lo == kLoEmpty) return a;
  if (a.lo == kLoEmpty) return b;
  if (a.flags | b.flags || big(a) || big(b)) return Summ{0, 0, 0, 1};
  return Summ{a.P + b.P, min(a.lo, a.P + b.lo), max(a.hi, a.P + b.hi), 0};
}

// A: bound = |s0| + sum |x| (double, atomics: only the window depends on it,
// never the result)
__global__ void xs_bound_kernel(const float *__restrict__ x, int64_t n, double *bound) {
  double a = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a += fabs((double)x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    a = threadIdx.x < blockDim.x / 32 ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) atomicAdd(bound, a);
  }
}

__device__ __forceinline__ int window_lo(const double *bound, float s0) {
  const double b = (*bound + fabs((double)s0)) * 1.0009765625 + 1e-30;
  int e;
  frexp(b, &e);  // b in [2^(e-1), 2^e); one binade of headroom above for
                 // the accumulated rounding of long sums
  return e - (XS_W - 1);
}

// B: chunk and super-chunk summaries for every window binade.  A warp owns a
// chunk; lane k (k < 16) runs binade elo + k over the first half of the
// chunk, lane 16 + k over the second half, and the halves are merged.
__global__ void __launch_bounds__(1024) xs_summ_kernel(const float *__restrict__ x, int64_t n, const double *bound,
                                                        float s0, Summ *__restrict__ chunks,
                                                        Summ *__restrict__ supers, int64_t nchunks) {
  __shared__ float xs[XS_SUPER][XS_CHUNK + 1];
  __shared__ Summ sm[XS_SUPER][XS_W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * XS_SUPER + warp;
  const int elo = window_lo(bound, s0);
  const int64_t base = c * XS_CHUNK;
  const int cnt = c < nchunks ? (int)min((int64_t)XS_CHUNK, n - base) : 0;
#pragma unroll
  for (int j = 0; j < XS_PER_LANE; ++j) {
    const int i = lane + 32 * j;
    xs[warp][i + (i >> 7)] = i < cnt ? x[base + i] : 0.f;  // halves in different banks
  }
  __syncwarp();
  const int k = lane & (XS_W - 1), h = lane >> 4;
  const int e = elo + k;
  int P = 0, lo = kLoEmpty, hi = kHiEmpty, flag = 0;
  const int i0 = h * (XS_CHUNK / 2), i1 = min(i0 + XS_CHUNK / 2, cnt);
  if (i1 - i0 == XS_CHUNK / 2) {
    // full half: 8 elements per step, loads first (independent of the scan)
#pragma unroll 2
    for (int i = i0; i < i1; i += 8) {
      uint32_t b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = __float_as_uint(xs[warp][i + j + h]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        P += units(b[j], e, flag);  // |P| < 128 * 2^24: no overflow
        lo = min(lo, P - 1);
        hi = max(hi, P + 1);
      }
    }
  } else {
    for (int i = i0; i < i1; ++i) {
      P += units(__float_as_uint(xs[warp][i + h]), e, flag);
      lo = min(lo, P - 1);
      hi = max(hi, P + 1);
    }
  }
  Summ s{P, lo, hi, flag};
  Summ t;
  t.P = __shfl_down_sync(0xffffffffu, s.P, 16);
  t.lo = __shfl_down_sync(0xffffffffu, s.lo, 16);
  t.hi = __shfl_down_sync(0xffffffffu, s.hi, 16);
  t.flags = __shfl_down_sync(0xffffffffu, s.flags, 16);
  if (lane < XS_W) {
    s = merge(s, t);
    if (c < nchunks) chunks[c * XS_W + k] = s;
    sm[warp][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < XS_W) {
    const int kk = threadIdx.x;
    Summ a = sm[0][kk];
    for (int w = 1; w < XS_SUPER; ++w) a = merge(a, sm[w][kk]);
    supers[(int64_t)blockIdx.x * XS_W + kk] = a;
  }
}

// apply the binade-k record of a summary row (row[k], k from s) to s.
// s < 0 runs the mirrored problem: fl(s + x) = -fl(|s| + (-x)), whose units
// are -r, so the prefix range flips (|S| - hi, |S| - lo) and S' = |S| - P.
__device__ __forceinline__ bool apply(float &s, const Summ *row, int elo) {
  const uint32_t bits = __float_as_uint(s);
  const uint32_t exr = (bits >> 23) & 0xFFu;
  const int k = (int)exr - 127 - elo;
  if (exr == 0 || exr == 0xFFu || k < 0 || k >= XS_W) return false;
  const Summ t = row[k];
  if (t.flags) return false;
  if (t.lo == kLoEmpty) return true;
  const int S = (int)((bits & 0x7FFFFFu) | 0x800000u);
  int S2;
  if ((bits >> 31) == 0) {
    if (S + t.lo < (1 << 23) || S + t.hi > (1 << 24)) return false;
    S2 = S + t.P;
  } else {
    if (S - t.hi < (1 << 23) || S - t.lo > (1 << 24)) return false;
    S2 = S - t.P;
  }
  s = __uint_as_float((bits & 0x80000000u) | (exr << 23) | (uint32_t)(S2 - (1 << 23)));
  return true;
}

// C: the serial walk (one warp).  Super-chunk summaries stream through a
// double-buffered shared-memory window of 32 super-chunks (the next window's
// loads are in flight while the current one is walked); a descent loads the
// 32 chunk summaries of one super-chunk at once.
__global__ void __launch_bounds__(32) xs_compose_kernel(const float *__restrict__ x, int64_t n,
                                                         const double *bound, float s0,
                                                         const Summ *__restrict__ chunks,
                                                         const Summ *__restrict__ supers, int64_t nchunks,
                                                         int64_t nsupers, float *out, int stats) {
  int n_desc = 0, n_slow = 0, n_super_ok = 0;
  constexpr int G = 32;                       // super-chunks per window
  constexpr int REC = G * XS_W;               // records per window (int4 each)
  __shared__ int4 sbuf[2][REC];
  __shared__ int4 cbuf[XS_SUPER * XS_W];
  __shared__ __align__(16) float xbuf[XS_CHUNK];
  const int lane = threadIdx.x;
  const int elo = window_lo(bound, s0);
  const int4 *sup4 = reinterpret_cast<const int4 *>(supers);
  const int4 *chk4 = reinterpret_cast<const int4 *>(chunks);
  const int64_t nrec = nsupers * XS_W;
  int4 pre[REC / 32];
  auto fetch = [&](int64_t g) {
#pragma unroll
    for (int j = 0; j < REC / 32; ++j) {
      const int64_t r = g * REC + lane + 32 * j;
      pre[j] = r < nrec ? sup4[r] : make_int4(0, 0, 0, 1);
    }
  };
  auto stash = [&](int b) {
#pragma unroll
    for (int j = 0; j < REC / 32; ++j) sbuf[b][lane + 32 * j] = pre[j];
  };
  float s = s0;
  const int64_t ngroups = (nsupers + G - 1) / G;
  fetch(0);
  stash(0);
  __syncwarp();
  for (int64_t g = 0; g < ngroups; ++g) {
    const int cur = (int)(g & 1);
    if (g + 1 < ngroups) fetch(g + 1);
    const int64_t s_end = min((g + 1) * G, nsupers);
    for (int64_t sc = g * G; sc < s_end; ++sc) {
      if (apply(s, reinterpret_cast<const Summ *>(&sbuf[cur][(sc - g * G) * XS_W]), elo)) {
        ++n_super_ok;
        continue;
      }
      ++n_desc;
      const int64_t c0 = sc * XS_SUPER, c1 = min(c0 + XS_SUPER, nchunks);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < XS_SUPER * XS_W / 32; ++j) {
        const int64_t r = c0 * XS_W + lane + 32 * j;
        cbuf[lane + 32 * j] = r < nchunks * XS_W ? chk4[r] : make_int4(0, 0, 0, 1);
      }
      __syncwarp();
      for (int64_t c = c0; c < c1; ++c) {
        if (apply(s, reinterpret_cast<const Summ *>(&cbuf[(c - c0) * XS_W]), elo)) continue;
        // element by element: the definition
        ++n_slow;
        const int64_t base = c * XS_CHUNK;
        const int cnt = (int)min((int64_t)XS_CHUNK, n - base);
#pragma unroll
        for (int j = 0; j < XS_PER_LANE; ++j) {
          const int i = lane + 32 * j;
          xbuf[i] = i < cnt ? x[base + i] : 0.f;
        }
        __syncwarp();
        if (lane == 0) {
          int i = 0;
          for (; i + 8 <= cnt; i += 8) {  // operands fetched ahead of the dependent adds
            const float4 a = *reinterpret_cast<const float4 *>(&xbuf[i]);
            const float4 b = *reinterpret_cast<const float4 *>(&xbuf[i + 4]);
            s = __fadd_rn(s, a.x); s = __fadd_rn(s, a.y); s = __fadd_rn(s, a.z); s = __fadd_rn(s, a.w);
            s = __fadd_rn(s, b.x); s = __fadd_rn(s, b.y); s = __fadd_rn(s, b.z); s = __fadd_rn(s, b.w);
          }
          for (; i < cnt; ++i) s = __fadd_rn(s, xbuf[i]);
        }
        s = __shfl_sync(0xffffffffu, s, 0);
        __syncwarp();
      }
    }
    __syncwarp();
    if (g + 1 < ngroups) stash(cur ^ 1);
    __syncwarp();
  }
  if (lane == 0) *out = s;
  if (stats && lane == 0)
    printf("[xsum] n=%lld supers=%lld ok=%d descents=%d slow_chunks=%d elo=%d\n", (long long)n,
           (long long)nsupers, n_super_ok, n_desc, n_slow, elo);
}

struct Workspace {
  void *p = nullptr;
  size_t bytes = 0;
};
std::mutex ws_mu;
std::map<int, Workspace> ws_by_dev;

}  // namespace

extern "C" size_t b2o_exact_sum_workspace(int64_t n) {
  const int64_t nchunks = (n + XS_CHUNK - 1) / XS_CHUNK;
  const int64_t nsupers = (nchunks + XS_SUPER - 1) / XS_SUPER;
  return 256 + sizeof(Summ) * XS_W * (size_t)(nchunks + nsupers + 32 * XS_W);
}

// s_out = (((s0 + x[0]) + x[1]) + ...) in fp32, bit-identical to the loop;
// workspace: device memory of b2o_exact_sum_workspace(n) bytes (NULL: an
// internal per-device buffer).  Asynchronous on `stream`.
extern "C" int b2o_exact_sum_f32_ws(const float *x, int64_t n, float s0, float *s_out, void *workspace,
                                    void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0) return -1;
  if (n == 0) {
    return cudaMemcpyAsync(s_out, &s0, sizeof(float), cudaMemcpyHostToDevice, st) == cudaSuccess ? 0 : -1;
  }
  const int64_t nchunks = (n + XS_CHUNK - 1) / XS_CHUNK;
  const int64_t nsupers = (nchunks + XS_SUPER - 1) / XS_SUPER;
  char *ws = (char *)workspace;
  double *bound = (double *)ws;
  Summ *chunks = (Summ *)(ws + 256);
  Summ *supers = chunks + XS_W * nchunks;
  if (cudaMemsetAsync(bound, 0, sizeof(double), st) != cudaSuccess) return -1;
  const int gb = (int)std::min<int64_t>(148 * 8, (n + 255) / 256);
  xs_bound_kernel<<<gb, 256, 0, st>>>(x, n, bound);
  xs_summ_kernel<<<(unsigned)nsupers, 1024, 0, st>>>(x, n, bound, s0, chunks, supers, nchunks);
  static const int stats = getenv("B2O_XSUM_STATS") != nullptr;
  xs_compose_kernel<<<1, 32, 0, st>>>(x, n, bound, s0, chunks, supers, nchunks, nsupers, s_out, stats);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int b2o_exact_sum_f32(const float *x, int64_t n, float s0, float *s_out, void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = b2o_exact_sum_workspace(n);
  void *ws = nullptr;
  {
    std::lock_guard<std::mutex> lk(ws_mu);
    Workspace &w = ws_by_dev[dev];
    if (w.bytes < need) {
      if (w.p) {
        cudaStreamSynchronize((cudaStream_t)stream);
        cudaFree(w.p);
      }
      w.p = nullptr;
      w.bytes = 0;
      if (cudaMalloc(&w.p, need) != cudaSuccess) return -1;
      w.bytes = need;
    }
    ws = w.p;
  }
  return b2o_exact_sum_f32_ws(x, n, s0, s_out, ws, stream);
}
