// b2o_xsum.cu — the sequential fp32 sum  s = s + x[0] + x[1] + ... (each
// addition rounded to fp32, in index order: the C loop `gosa = gosa + gs[i]`)
// computed in parallel on the GPU, bit-identical to the sequential loop.
//
// Why it parallelises: while the running sum s stays inside one binade
// [2^e, 2^(e+1)) it is an integer S in units u = 2^(e-23), S in [2^23, 2^24),
// and
//
//     fl(s + x) = (S + r) u,   r = round-to-nearest(x / u),
//
// provided the exact sum stays inside the binade.  r depends on x and e only
// -- except for an x exactly half-way between two multiples of u, which
// rounds to the even neighbour: r = floor(x / u) + parity(S + floor(x / u)),
// after which S is even.  So for a fixed binade the effect of a run of
// elements is, for each parity of S at its start, an integer sum plus the
// range of the running integer prefix (to check that s never left the
// binade); runs compose associatively (the first run's end parity selects
// the second's variant), hence scan-ably.  Every element's validity
// condition is kept conservative:
//
//     S + P_j + r_j - 1 >= 2^23   and   S + P_j + r_j + 1 <= 2^24
//
// (P_j = r_0 + ... + r_(j-1)); an infinity / NaN or an x too large for the
// binade flags the run as unusable.
//
// Four kernels on the caller's stream:
//   A  stats:    per super-chunk (8192 terms) its sum and its reach (extreme
//                chunk-boundary prefixes + the largest chunk magnitude);
//   A2 window:   one CTA scans the sums: each super-chunk gets the 4 binades
//                below (|s0 + earlier sums| + its reach) * 1.25;
//   B  summarise: per chunk of 256 terms (one warp: 8 parts x 4 binades) and
//                per super-chunk: (P, min prefix - 1, max prefix + 1) for
//                both start parities, and flags, for each window binade;
//   C  compose:  one warp walks the super-chunks 32 at a time: lane i picks
//                super-chunk i's record for the running sum's binade, a warp
//                scan merges them in order and the longest usable prefix is
//                applied in O(1); a super-chunk that is not usable is walked
//                by its chunks the same way, and a chunk that is not usable
//                either (a binade crossing, a running sum outside the window
//                or not normal) is added element by element with __fadd_rn --
//                the definition itself.
// Himeno M's 4.1 M gosa terms: 0.15 ms (10 descents, 16 element-wise chunks).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <map>

#include "../../include/b2o.h"

namespace {

constexpr int XS_CHUNK = 256;        // elements per chunk (one warp, 8 per lane)
constexpr int XS_PER_LANE = XS_CHUNK / 32;
constexpr int XS_SUPER = 32;         // chunks per super-chunk (one CTA of 32 warps)
constexpr int XS_W = 4;              // binades in each super-chunk's window

// The two IEEE formats: value type, raw bits, the signed integer that holds a
// run's increments, the fraction width and exponent field.
struct F32 {
  using V = float;
  using U = uint32_t;
  using I = int;
  static constexpr int MANT = 23, EMASK = 0xFF, BIAS = 127;
  static constexpr I kLoEmpty = 0x7FFFFFFF, kHiEmpty = -0x7FFFFFFF - 1, kBig = 1 << 25;
  static __device__ __forceinline__ U bits(V v) { return __float_as_uint(v); }
  static __device__ __forceinline__ V value(U b) { return __uint_as_float(b); }
  static __device__ __forceinline__ V add(V a, V b) { return __fadd_rn(a, b); }
};
struct F64 {
  using V = double;
  using U = unsigned long long;
  using I = long long;
  static constexpr int MANT = 52, EMASK = 0x7FF, BIAS = 1023;
  static constexpr I kLoEmpty = 0x7FFFFFFFFFFFFFFFLL, kHiEmpty = -0x7FFFFFFFFFFFFFFFLL - 1, kBig = 1LL << 54;
  static __device__ __forceinline__ U bits(V v) { return (U)__double_as_longlong(v); }
  static __device__ __forceinline__ V value(U b) { return __longlong_as_double((long long)b); }
  static __device__ __forceinline__ V add(V a, V b) { return __dadd_rn(a, b); }
};

// A run's effect for one binade, in units u, for both parities of the
// running integer S at the run's start (variant p: S odd iff p = 1): a term
// exactly half-way between two multiples of u rounds to the even neighbour,
// so its increment depends on the parity of S there -- and after it S is
// even, whichever way it went.  Tracking both start parities keeps ties on
// the fast path; merging runs maps each start parity through the first run's
// end parity.  Valid summaries have |P|, |lo|, |hi| <= 2^(MANT+1) + 1 (the
// running integer stays in [2^MANT, 2^(MANT+1))); larger ones are flagged,
// which also keeps every integer sum below overflow.
template <class T>
struct alignas(16) Summ {
  typename T::I P0, P1;    // sum of the increments
  typename T::I lo0, lo1;  // min over j of (P_(j+1) - 1)
  typename T::I hi0, hi1;  // max over j of (P_(j+1) + 1)
  int flags;               // nonzero: unusable for this binade
  int pad;
};

template <class T>
__device__ __forceinline__ Summ<T> empty_summ() {
  return Summ<T>{0, 0, T::kLoEmpty, T::kLoEmpty, T::kHiEmpty, T::kHiEmpty, 0, 0};
}
template <class T>
__device__ __forceinline__ Summ<T> invalid_summ() {
  return Summ<T>{0, 0, 0, 0, 0, 0, 1, 0};
}

// x / 2^(e-MANT) rounded to nearest, as raw bits: returns round(X) (tie = 0)
// or floor(X) for a half-way X (tie = 1; the increment is floor(X) + the
// parity of S + floor(X)).  Branch-free (the lanes of a warp evaluate
// different binades).  |x| >= 2^(e+1) (d > 0) can never keep the sum in the
// binade and inf / nan are flagged.
template <class T>
__device__ __forceinline__ typename T::I units(typename T::U bits, int e, int &tie, int &flag) {
  using U = typename T::U;
  using I = typename T::I;
  constexpr int W = 8 * (int)sizeof(U);
  const int exr = (int)((bits >> T::MANT) & (U)T::EMASK);
  const U m = (bits & (((U)1 << T::MANT) - 1)) | (exr ? ((U)1 << T::MANT) : (U)0);
  const int ex = exr ? exr - T::BIAS : 1 - T::BIAS;
  const int d = ex - e;
  const int sh = min(max(-d, 1), W - 1);
  const U q = m >> sh, rem = m & (((U)1 << sh) - 1), half = (U)1 << (sh - 1);
  flag |= (exr == T::EMASK) | (d > 0);
  const bool neg = (bits >> (W - 1)) != 0;
  tie = (d < 0 && rem == half) ? 1 : 0;
  if (tie) return neg ? -(I)q - 1 : (I)q;  // floor(X)
  const I r = d == 0 ? (I)m : (d < 0 ? (I)q + (rem > half ? 1 : 0) : 0);
  return neg ? -r : r;
}

// apply one term (c, tie) to both variants
template <class T>
__device__ __forceinline__ void step(Summ<T> &s, typename T::I c, int tie) {
  using I = typename T::I;
  const I r0 = c + ((I)tie & (s.P0 + c)), r1 = c + ((I)tie & (1 + s.P1 + c));
  s.P0 += r0;
  s.P1 += r1;
  s.lo0 = min(s.lo0, s.P0 - 1);
  s.hi0 = max(s.hi0, s.P0 + 1);
  s.lo1 = min(s.lo1, s.P1 - 1);
  s.hi1 = max(s.hi1, s.P1 + 1);
}

template <class T>
__device__ __forceinline__ bool big(const Summ<T> &a) {
  auto out = [](typename T::I v) { return v > T::kBig || v < -T::kBig; };
  return out(a.P0) || out(a.P1) || out(a.lo0) || out(a.lo1) || out(a.hi0) || out(a.hi1);
}

// a then b: variant p of a ends with parity (p + a.P_p) & 1, which selects b's
template <class T>
__device__ __forceinline__ Summ<T> merge(const Summ<T> &a, const Summ<T> &b) {
  using I = typename T::I;
  if (b.lo0 == T::kLoEmpty) return a;
  if (a.lo0 == T::kLoEmpty) return b;
  if (a.flags | b.flags || big<T>(a) || big<T>(b)) return invalid_summ<T>();
  const bool x0 = (a.P0 & 1) != 0, x1 = ((1 + a.P1) & 1) != 0;
  const I bP0 = x0 ? b.P1 : b.P0, bl0 = x0 ? b.lo1 : b.lo0, bh0 = x0 ? b.hi1 : b.hi0;
  const I bP1 = x1 ? b.P1 : b.P0, bl1 = x1 ? b.lo1 : b.lo0, bh1 = x1 ? b.hi1 : b.hi0;
  return Summ<T>{a.P0 + bP0, a.P1 + bP1, min(a.lo0, a.P0 + bl0), min(a.lo1, a.P1 + bl1),
                 max(a.hi0, a.P0 + bh0), max(a.hi1, a.P1 + bh1), 0, 0};
}

template <class T>
__device__ __forceinline__ Summ<T> shfl_down_summ(const Summ<T> &s, int d) {
  return Summ<T>{__shfl_down_sync(0xffffffffu, s.P0, d), __shfl_down_sync(0xffffffffu, s.P1, d),
                 __shfl_down_sync(0xffffffffu, s.lo0, d), __shfl_down_sync(0xffffffffu, s.lo1, d),
                 __shfl_down_sync(0xffffffffu, s.hi0, d), __shfl_down_sync(0xffffffffu, s.hi1, d),
                 __shfl_down_sync(0xffffffffu, s.flags, d), 0};
}

template <class T>
__device__ __forceinline__ Summ<T> shfl_up_summ(const Summ<T> &s, int d) {
  return Summ<T>{__shfl_up_sync(0xffffffffu, s.P0, d), __shfl_up_sync(0xffffffffu, s.P1, d),
                 __shfl_up_sync(0xffffffffu, s.lo0, d), __shfl_up_sync(0xffffffffu, s.lo1, d),
                 __shfl_up_sync(0xffffffffu, s.hi0, d), __shfl_up_sync(0xffffffffu, s.hi1, d),
                 __shfl_up_sync(0xffffffffu, s.flags, d), 0};
}

template <class T>
__device__ __forceinline__ Summ<T> shfl_summ(const Summ<T> &s, int src) {
  return Summ<T>{__shfl_sync(0xffffffffu, s.P0, src), __shfl_sync(0xffffffffu, s.P1, src),
                 __shfl_sync(0xffffffffu, s.lo0, src), __shfl_sync(0xffffffffu, s.lo1, src),
                 __shfl_sync(0xffffffffu, s.hi0, src), __shfl_sync(0xffffffffu, s.hi1, src),
                 __shfl_sync(0xffffffffu, s.flags, src), 0};
}

// A: per super-chunk (double): its sum, and how far the running sum can get
// from the super-chunk's starting value: the extreme prefix sums at chunk
// boundaries plus the largest chunk magnitude (a chunk's own excursion)
template <class T>
__global__ void __launch_bounds__(256) xs_stats_kernel(const typename T::V *__restrict__ x, int64_t n,
                                                        double *__restrict__ ssum, double *__restrict__ sreach) {
  __shared__ double cs[XS_SUPER], ca[XS_SUPER];
  const int64_t b0 = (int64_t)blockIdx.x * XS_SUPER * XS_CHUNK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < XS_SUPER; c += blockDim.x / 32) {
    double a = 0.0, m = 0.0;
    for (int i = lane; i < XS_CHUNK; i += 32) {
      const int64_t g = b0 + (int64_t)c * XS_CHUNK + i;
      if (g < n) {
        const double v = (double)x[g];
        a += v;
        m += fabs(v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if (lane == 0) {
      cs[c] = a;
      ca[c] = m;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double pre = 0.0, lo = 0.0, hi = 0.0, am = 0.0;
    for (int c = 0; c < XS_SUPER; ++c) {
      pre += cs[c];
      lo = fmin(lo, pre);
      hi = fmax(hi, pre);
      am = fmax(am, ca[c]);
    }
    ssum[blockIdx.x] = pre;
    // reach: (lo, hi, chunk magnitude) packed as three doubles
    sreach[3 * blockIdx.x] = lo;
    sreach[3 * blockIdx.x + 1] = hi;
    sreach[3 * blockIdx.x + 2] = am;
  }
}

// A2: each super-chunk's binade window.  est = s0 + sum of the earlier
// super-chunks (double); |s| inside the super-chunk is at most
// max(|est + lo|, |est + hi|) + the largest chunk magnitude, with 25 % slack
// for the drift of the running sum from the exact one; the window is the
// XS_W binades up to that bound (a running sum below it is added element by
// element: exact, only slower).
__global__ void __launch_bounds__(1024) xs_window_kernel(const double *__restrict__ ssum,
                                                          const double *__restrict__ sreach, int64_t nsupers,
                                                          double s0, int *__restrict__ ebase) {
  __shared__ double part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nsupers + 1023) / 1024;
  const int64_t i0 = t * per, i1 = min(i0 + per, nsupers);
  double loc = 0.0;
  for (int64_t i = i0; i < i1; ++i) loc += ssum[i];
  part[t] = loc;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // inclusive Hillis-Steele scan
    const double v = t >= d ? part[t - d] : 0.0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  double est = s0 + (t > 0 ? part[t - 1] : 0.0);
  for (int64_t i = i0; i < i1; ++i) {
    const double reach = fmax(fabs(est + sreach[3 * i]), fabs(est + sreach[3 * i + 1])) + sreach[3 * i + 2];
    const double top = reach * 1.25 + 1e-300;
    int e;
    frexp(top, &e);  // top in [2^(e-1), 2^e)
    ebase[i] = (e - 1) - (XS_W - 1);
    est += ssum[i];
  }
}

// B: chunk and super-chunk summaries for the XS_W window binades of their
// super-chunk.  A warp owns a chunk: lane = 4 * part + k runs binade
// ebase + k over part (32 elements) of the chunk; the 8 parts are merged in
// order with three shuffles.  The chunk is staged in (dynamic) shared memory.
template <class T>
__global__ void __launch_bounds__(1024) xs_summ_kernel(const typename T::V *__restrict__ x, int64_t n,
                                                        const int *__restrict__ ebase, Summ<T> *__restrict__ chunks,
                                                        Summ<T> *__restrict__ supers, int64_t nchunks) {
  using V = typename T::V;
  using I = typename T::I;
  constexpr int ROW = XS_CHUNK + XS_CHUNK / 32;
  extern __shared__ __align__(16) unsigned char xs_raw[];
  V *xs = reinterpret_cast<V *>(xs_raw);
  __shared__ Summ<T> sm[XS_SUPER][XS_W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * XS_SUPER + warp;
  const int64_t base = c * XS_CHUNK;
  const int cnt = c < nchunks ? (int)min((int64_t)XS_CHUNK, n - base) : 0;
  V *my = xs + warp * ROW;
#pragma unroll
  for (int j = 0; j < XS_PER_LANE; ++j) {
    const int i = lane + 32 * j;
    my[i + (i >> 5)] = i < cnt ? x[base + i] : (V)0;  // parts in different banks
  }
  __syncwarp();
  const int k = lane & (XS_W - 1), part = lane >> 2;
  const int e = ebase[blockIdx.x] + k;
  constexpr int PART = XS_CHUNK / 8;
  Summ<T> s = empty_summ<T>();
  int flag = 0;
  const int i0 = part * PART, i1 = min(i0 + PART, cnt);
  const V *row = my + part * (PART + 1);
  if (i1 - i0 == PART) {
#pragma unroll 4
    for (int i = 0; i < PART; i += 8) {
      typename T::U b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = T::bits(row[i + j]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int tie;
        const I cc = units<T>(b[j], e, tie, flag);  // |P| < 32 * 2^(MANT+1): no overflow
        step<T>(s, cc, tie);
      }
    }
  } else {
    for (int i = 0; i < i1 - i0; ++i) {
      int tie;
      const I cc = units<T>(T::bits(row[i]), e, tie, flag);
      step<T>(s, cc, tie);
    }
  }
  s.flags = flag;
#pragma unroll
  for (int d = 4; d < 32; d <<= 1) {  // ordered merge: part p with part p + d/4
    const Summ<T> t = shfl_down_summ<T>(s, d);
    if ((part & (2 * (d >> 2) - 1)) == 0) s = merge<T>(s, t);
  }
  if (lane < XS_W) {
    if (c < nchunks) chunks[c * XS_W + k] = s;
    sm[warp][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < XS_W) {
    const int kk = threadIdx.x;
    Summ<T> a = sm[0][kk];
    for (int w = 1; w < XS_SUPER; ++w) a = merge<T>(a, sm[w][kk]);
    supers[(int64_t)blockIdx.x * XS_W + kk] = a;
  }
}

// ---- C: the in-order walk (one warp) -------------------------------------

template <class T>
struct WalkState {
  bool ok;            // s is a normal number
  int e;              // its binade: |s| in [2^e, 2^(e+1))
  typename T::I S;    // |s| / 2^(e-MANT), in [2^MANT, 2^(MANT+1))
  bool neg;
};

template <class T>
__device__ __forceinline__ WalkState<T> state_of(typename T::V s) {
  using U = typename T::U;
  const U b = T::bits(s);
  const int exr = (int)((b >> T::MANT) & (U)T::EMASK);
  return WalkState<T>{exr != 0 && exr != T::EMASK, exr - T::BIAS,
                      (typename T::I)((b & (((U)1 << T::MANT) - 1)) | ((U)1 << T::MANT)),
                      (b >> (8 * sizeof(U) - 1)) != 0};
}

// a run summary (for s's binade) is usable from state w: the variant of S's
// parity.  s < 0 runs the mirrored problem fl(s + x) = -fl(|s| + (-x)): the
// increments negate (ties included, round-half-even being symmetric) and the
// parity evolution is the same, so the prefix range flips (|S| - hi,
// |S| - lo) and S' = |S| - P.
template <class T>
__device__ __forceinline__ bool usable(const Summ<T> &t, const WalkState<T> &w) {
  using I = typename T::I;
  constexpr I lo_lim = (I)1 << T::MANT, hi_lim = (I)1 << (T::MANT + 1);
  if (t.flags) return false;
  if (t.lo0 == T::kLoEmpty) return true;
  const bool odd = (w.S & 1) != 0;
  const I lo = odd ? t.lo1 : t.lo0, hi = odd ? t.hi1 : t.hi0;
  return w.neg ? (w.S - hi >= lo_lim && w.S - lo <= hi_lim) : (w.S + lo >= lo_lim && w.S + hi <= hi_lim);
}

template <class T>
__device__ __forceinline__ typename T::V advance(typename T::V s, const Summ<T> &t, const WalkState<T> &w) {
  using U = typename T::U;
  using I = typename T::I;
  if (t.lo0 == T::kLoEmpty) return s;
  const I P = (w.S & 1) ? t.P1 : t.P0;
  const I S2 = w.neg ? w.S - P : w.S + P;
  const U keep = ~(((U)1 << T::MANT) - 1);  // sign and exponent
  return T::value((T::bits(s) & keep) | (U)(S2 - ((I)1 << T::MANT)));
}

// lane i holds the summary (for s's binade) of run i: empty outside
// [first, cnt), invalid when its window lacks the binade.  Applies the
// longest usable prefix of runs first.. to s; returns how many runs that was.
template <class T>
__device__ __forceinline__ int scan_apply(typename T::V &s, Summ<T> mine, int first, int cnt,
                                          const WalkState<T> &w) {
  const int lane = threadIdx.x & 31;
  Summ<T> pre = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Summ<T> t = shfl_up_summ<T>(pre, d);
    if (lane >= d) pre = merge<T>(t, pre);
  }
  const unsigned bad = __ballot_sync(0xffffffffu, lane >= first && lane < cnt && !usable<T>(pre, w));
  const int f = bad ? __ffs(bad) - 1 : cnt;
  if (f > first) s = advance<T>(s, shfl_summ<T>(pre, f - 1), w);
  return f - first;
}

// C: one warp walks the super-chunks 32 at a time: lane i picks super-chunk
// i's record for s's binade, a warp scan merges them in order and the
// longest usable prefix is applied in O(1).  A super-chunk that is not
// usable is walked by its 32 chunks the same way; a chunk that is not usable
// either (binade crossing, s outside its window or not normal) is added
// element by element with a correctly rounded add -- the definition.  The
// next group's records are loaded while the current group is walked.
template <class T>
__global__ void __launch_bounds__(32) xs_compose_kernel(const typename T::V *__restrict__ x, int64_t n,
                                                         const int *__restrict__ ebase, typename T::V s0,
                                                         const Summ<T> *__restrict__ chunks,
                                                         const Summ<T> *__restrict__ supers, int64_t nchunks,
                                                         int64_t nsupers, typename T::V *out, int stats) {
  using V = typename T::V;
  constexpr int R4 = (int)(sizeof(Summ<T>) / sizeof(int4));  // int4 per record
  __shared__ int4 sbuf[2][32 * XS_W * R4];
  __shared__ int4 cbuf[XS_SUPER * XS_W * R4];
  __shared__ __align__(16) V xbuf[XS_CHUNK];
  const int lane = threadIdx.x;
  const int4 *sup4 = reinterpret_cast<const int4 *>(supers);
  const int4 *chk4 = reinterpret_cast<const int4 *>(chunks);
  int n_desc = 0, n_slow = 0;
  int4 pre[XS_W * R4];
  int peb = 0;
  auto fetch = [&](int64_t g) {
#pragma unroll
    for (int j = 0; j < XS_W * R4; ++j) {
      const int64_t r = g * 32 * XS_W * R4 + lane + 32 * j;
      pre[j] = r < nsupers * XS_W * R4 ? sup4[r] : make_int4(0, 0, 0, 0);
    }
    peb = g * 32 + lane < nsupers ? ebase[g * 32 + lane] : 0;
  };
  auto stash = [&](int b) {
#pragma unroll
    for (int j = 0; j < XS_W * R4; ++j) sbuf[b][lane + 32 * j] = pre[j];
  };
  V s = s0;
  const int64_t ngroups = (nsupers + 31) / 32;
  fetch(0);
  stash(0);
  int eb = peb;
  __syncwarp();
  for (int64_t g = 0; g < ngroups; ++g) {
    const int cur = (int)(g & 1);
    if (g + 1 < ngroups) fetch(g + 1);
    const int cnt = (int)min((int64_t)32, nsupers - g * 32);
    const Summ<T> *srec = reinterpret_cast<const Summ<T> *>(sbuf[cur]);
    int pos = 0;
    while (pos < cnt) {
      WalkState<T> w = state_of<T>(s);
      if (w.ok) {
        const int k = w.e - eb;
        Summ<T> mine = (lane < pos || lane >= cnt)
                           ? empty_summ<T>()
                           : ((k >= 0 && k < XS_W) ? srec[lane * XS_W + k] : invalid_summ<T>());
        pos += scan_apply<T>(s, mine, pos, cnt, w);
        if (pos >= cnt) break;
      }
      // super-chunk g*32 + pos by its chunks
      ++n_desc;
      const int64_t sc = g * 32 + pos;
      const int ceb = __shfl_sync(0xffffffffu, eb, pos);
      const int64_t c0 = sc * XS_SUPER, c1 = min(c0 + XS_SUPER, nchunks);
      const int nc = (int)(c1 - c0);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < XS_W * R4; ++j) {
        const int64_t r = c0 * XS_W * R4 + lane + 32 * j;
        cbuf[lane + 32 * j] = r < nchunks * XS_W * R4 ? chk4[r] : make_int4(0, 0, 0, 0);
      }
      __syncwarp();
      const Summ<T> *crec = reinterpret_cast<const Summ<T> *>(cbuf);
      int cpos = 0;
      while (cpos < nc) {
        w = state_of<T>(s);
        if (w.ok) {
          const int k = w.e - ceb;
          Summ<T> mine = (lane < cpos || lane >= nc)
                             ? empty_summ<T>()
                             : ((k >= 0 && k < XS_W) ? crec[lane * XS_W + k] : invalid_summ<T>());
          cpos += scan_apply<T>(s, mine, cpos, nc, w);
          if (cpos >= nc) break;
        }
        // chunk c0 + cpos element by element
        ++n_slow;
        const int64_t base = (c0 + cpos) * XS_CHUNK;
        const int m = (int)min((int64_t)XS_CHUNK, n - base);
#pragma unroll
        for (int j = 0; j < XS_PER_LANE; ++j) {
          const int i = lane + 32 * j;
          xbuf[i] = i < m ? x[base + i] : (V)0;
        }
        __syncwarp();
        if (lane == 0) {
          int i = 0;
          for (; i + 8 <= m; i += 8) {  // operands fetched ahead of the dependent adds
            V v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = xbuf[i + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) s = T::add(s, v[j]);
          }
          for (; i < m; ++i) s = T::add(s, xbuf[i]);
        }
        s = __shfl_sync(0xffffffffu, s, 0);
        __syncwarp();
        ++cpos;
      }
      ++pos;
    }
    __syncwarp();
    if (g + 1 < ngroups) {
      stash(cur ^ 1);
      eb = peb;
    }
    __syncwarp();
  }
  if (lane == 0) *out = s;
  if (stats && lane == 0)
    printf("[xsum] n=%lld supers=%lld descents=%d slow_chunks=%d\n", (long long)n, (long long)nsupers, n_desc,
           n_slow);
}

struct Workspace {
  void *p = nullptr;
  size_t bytes = 0;
};
std::mutex ws_mu;
std::map<int, Workspace> ws_by_dev;
std::atomic<bool> g_attr[2][64];  // per (format, device) smem attribute set (cleared on device reset)

struct Layout {
  int64_t nchunks, nsupers;
  size_t ssum, sreach, ebase, chunks, supers, bytes;
};

template <class T>
Layout layout(int64_t n) {
  Layout L;
  L.nchunks = (n + XS_CHUNK - 1) / XS_CHUNK;
  L.nsupers = (L.nchunks + XS_SUPER - 1) / XS_SUPER;
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  L.ssum = 0;
  L.sreach = up(L.ssum + sizeof(double) * L.nsupers);  // (lo, hi, chunk magnitude) per super-chunk
  L.ebase = up(L.sreach + 3 * sizeof(double) * L.nsupers);
  L.chunks = up(L.ebase + sizeof(int) * (L.nsupers + 32));
  L.supers = up(L.chunks + sizeof(Summ<T>) * XS_W * L.nchunks);
  L.bytes = up(L.supers + sizeof(Summ<T>) * XS_W * (L.nsupers + 32));
  return L;
}

template <class T>
int exact_sum_ws(const typename T::V *x, int64_t n, typename T::V s0, typename T::V *s_out, void *workspace,
                 void *stream) {
  using V = typename T::V;
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0) return -1;
  if (n == 0) {
    static_assert(sizeof(V) <= 8, "");
    return cudaMemcpyAsync(s_out, &s0, sizeof(V), cudaMemcpyHostToDevice, st) == cudaSuccess ? 0 : -1;
  }
  const Layout L = layout<T>(n);
  char *ws = (char *)workspace;
  double *ssum = (double *)(ws + L.ssum), *sreach = (double *)(ws + L.sreach);
  int *ebase = (int *)(ws + L.ebase);
  Summ<T> *chunks = (Summ<T> *)(ws + L.chunks), *supers = (Summ<T> *)(ws + L.supers);
  constexpr int kSummSmem = XS_SUPER * (XS_CHUNK + XS_CHUNK / 32) * (int)sizeof(V);
  std::atomic<bool> *attr = g_attr[sizeof(typename T::V) == 8];
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    if (cudaFuncSetAttribute(xs_summ_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSummSmem) !=
        cudaSuccess)
      return -1;
    attr[dev & 63] = true;
  }
  xs_stats_kernel<T><<<(unsigned)L.nsupers, 256, 0, st>>>(x, n, ssum, sreach);
  xs_window_kernel<<<1, 1024, 0, st>>>(ssum, sreach, L.nsupers, (double)s0, ebase);
  xs_summ_kernel<T><<<(unsigned)L.nsupers, 1024, kSummSmem, st>>>(x, n, ebase, chunks, supers, L.nchunks);
  static const int stats = getenv("B2O_XSUM_STATS") != nullptr;
  xs_compose_kernel<T><<<1, 32, 0, st>>>(x, n, ebase, s0, chunks, supers, L.nchunks, L.nsupers, s_out, stats);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <class T>
int exact_sum(const typename T::V *x, int64_t n, typename T::V s0, typename T::V *s_out, void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = layout<T>(std::max<int64_t>(n, 1)).bytes;
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
  return exact_sum_ws<T>(x, n, s0, s_out, ws, stream);
}

}  // namespace

// workspace bytes for either format (the fp64 records are the larger)
extern "C" size_t b2o_exact_sum_workspace(int64_t n) { return layout<F64>(std::max<int64_t>(n, 1)).bytes; }

// s_out = (((s0 + x[0]) + x[1]) + ...), each addition rounded to the format,
// bit-identical to the loop; workspace: device memory of
// b2o_exact_sum_workspace(n) bytes.  Asynchronous on `stream`.
extern "C" int b2o_exact_sum_f32_ws(const float *x, int64_t n, float s0, float *s_out, void *workspace,
                                    void *stream) {
  return exact_sum_ws<F32>(x, n, s0, s_out, workspace, stream);
}

extern "C" int b2o_exact_sum_f64_ws(const double *x, int64_t n, double s0, double *s_out, void *workspace,
                                    void *stream) {
  return exact_sum_ws<F64>(x, n, s0, s_out, workspace, stream);
}

extern "C" int b2o_exact_sum_f32(const float *x, int64_t n, float s0, float *s_out, void *stream) {
  return exact_sum<F32>(x, n, s0, s_out, stream);
}

extern "C" int b2o_exact_sum_f64(const double *x, int64_t n, double s0, double *s_out, void *stream) {
  return exact_sum<F64>(x, n, s0, s_out, stream);
}

// force-load this file's kernels (lazy module loading would otherwise charge
// the first timed pattern that uses one); called per device by b2o_init
// the device was reset (runtime broken-worker recovery): drop its workspace
// and attribute flags
extern "C" void b2o_xsum_forget_device(int dev) {
  std::lock_guard<std::mutex> lk(ws_mu);
  ws_by_dev.erase(dev);
  g_attr[0][dev & 63] = false;
  g_attr[1][dev & 63] = false;
}

extern "C" void b2o_xsum_warm(void) {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, xs_stats_kernel<F32>);
  cudaFuncGetAttributes(&a, xs_stats_kernel<F64>);
  cudaFuncGetAttributes(&a, xs_window_kernel);
  cudaFuncGetAttributes(&a, xs_summ_kernel<F32>);
  cudaFuncGetAttributes(&a, xs_summ_kernel<F64>);
  cudaFuncGetAttributes(&a, xs_compose_kernel<F32>);
  cudaFuncGetAttributes(&a, xs_compose_kernel<F64>);
  cudaGetLastError();
}
