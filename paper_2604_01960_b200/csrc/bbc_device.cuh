// Device helpers of the BBC query path: ordered float keys, block reductions/scans, and the
// CTA-wide radix select used for the probe top-nprobe, the sample's budget-th estimate
// (d_max) and the final top-k by (exact d^2, id) (Collect l.22-23).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

namespace bbc {

// BBC_CHECKS=1 (a test build, tests/test_bounds_checks.py): device-side bounds checks on the
// indices the scan, its ordering kernels, the compaction and the selections compute; a violation
// traps (the search then fails with a CUDA error).  compute-sanitizer is not available on the
// GPU pool, so this build plus the parity suite stands in for memcheck on these kernels.
#ifndef BBC_CHECKS
#define BBC_CHECKS 0
#endif
#define BBC_CHECK(cond)                                                                          \
  do {                                                                                           \
    if (BBC_CHECKS && !(cond)) {                                                                 \
      printf("BBC_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,      \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)

constexpr int kNStats = 7;          // device counters of a search (bbc_stats_vector)
constexpr int kCells = 256;          // 255 regular cells + overflow cell 255 (DESIGN R3)
constexpr int kTauInf = 1 << 30;     // tau = infinity (Alg. 1 l.11)
constexpr int kSampleMinLists = 8;   // "5-10 nearest clusters", DESIGN R5

// Monotone map float -> uint32 (total order of finite floats; -0 sorts before +0).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t shr64(uint64_t x, int s) { return s >= 64 ? 0ull : (x >> s); }

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp-aggregated shared-memory histogram update (north_star: "the bucket histogram uses
// warp-aggregated shared-memory atomics"): all 32 lanes call it with their bucket id (255 = beyond
// d_max, not counted); the lanes holding the same id are found with one match, and one of them
// adds their number -- one atomic per distinct id per warp instead of one per object.
__device__ __forceinline__ void warp_hist_add(int* hist, int cell) {
  const unsigned act = __ballot_sync(0xffffffffu, cell < 255);
  if (cell < 255) {
    const unsigned peers = __match_any_sync(act, cell);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[cell], __popc(peers));
  }
}

// Block-wide min and max of a 64-bit key; result broadcast to all threads.  `red` needs
// 2 * (NT/32) slots.
template <int NT>
__device__ __forceinline__ void block_minmax(uint64_t& mn, uint64_t& mx, uint64_t* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  mn = warp_min(mn);
  mx = warp_max(mx);
  if (lane == 0) { red[wid] = mn; red[NT / 32 + wid] = mx; }
  __syncthreads();
  if (wid == 0) {
    uint64_t a = lane < NT / 32 ? red[lane] : ~0ull;
    uint64_t b = lane < NT / 32 ? red[NT / 32 + lane] : 0ull;
    a = warp_min(a);
    b = warp_max(b);
    if (lane == 0) { red[0] = a; red[1] = b; }
  }
  __syncthreads();
  mn = red[0];
  mx = red[1];
  __syncthreads();
}

// Exclusive rank of a flagged thread among flagged threads in thread order; *total = count.
// `wcnt` needs NT/32 + 1 ints.  All threads must call.
template <int NT>
__device__ __forceinline__ int block_rank(bool flag, int* wcnt, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned b = __ballot_sync(0xffffffffu, flag);
  int inwarp = __popc(b & ((1u << lane) - 1u));
  if (lane == 0) wcnt[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    int v = lane < NT / 32 ? wcnt[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < NT / 32) wcnt[lane] = incl - v;
    if (lane == 31) wcnt[NT / 32] = incl;
  }
  __syncthreads();
  int r = wcnt[wid] + inwarp;
  *total = wcnt[NT / 32];
  __syncthreads();
  return r;
}

struct SelectSmem {
  unsigned hist[256];
  uint64_t red[64];
  uint64_t prefix;
  int pshift;
  int digit;
  long long need;
  unsigned cnt;
  int done;
};

// CTA-wide radix select over n 64-bit keys produced by load(i).
//   value_mode: returns the kth smallest key (duplicates allowed), *pshift = 0.
//   set mode (keys must be unique): returns (prefix, *pshift) such that exactly kth keys satisfy
//   shr64(key, *pshift) <= prefix.
// Passes of <= 8 bits from the highest bit where the minimum and maximum keys differ.
// An upper bound of the kth smallest key: the selection above stopped after `passes` digit
// passes, returning the largest key of the digit bin that holds the kth smallest (every key below
// it is in a lower bin).  At least the kth smallest key, at most that bin's last key.
template <int NT, typename LoadF>
__device__ uint64_t cta_select_upper(int64_t n, int64_t kth, LoadF load, int passes, SelectSmem& sm);

template <int NT, typename LoadF>
__device__ uint64_t cta_select(int64_t n, int64_t kth, LoadF load, bool value_mode, int* pshift_out,
                               SelectSmem& sm, int max_passes = 64) {
  uint64_t mn = ~0ull, mx = 0ull;
  for (int64_t i = threadIdx.x; i < n; i += NT) {
    uint64_t k = load(i);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  block_minmax<NT>(mn, mx, sm.red);
  if (mn == mx || kth <= 1) {
    *pshift_out = 0;
    if (mn == mx) return mn;
    if (kth <= 1) return mn;
  }
  const int bit = 63 - __clzll((long long)(mn ^ mx));
  int pshift = bit + 1;
  uint64_t prefix = shr64(mn, pshift);
  int shift = bit - 7 > 0 ? bit - 7 : 0;
  long long need = kth;
  while (true) {
    const int width = pshift - shift;
    const unsigned mask = (1u << width) - 1u;
    for (int i = threadIdx.x; i < 256; i += NT) sm.hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += NT) {
      uint64_t k = load(i);
      if (shr64(k, pshift) == prefix) atomicAdd(&sm.hist[(unsigned)(k >> shift) & mask], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned v[8];
      unsigned s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { v[j] = sm.hist[lane * 8 + j]; s += v[j]; }
      unsigned incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      unsigned excl = incl - s;
      // the lane whose range [excl, incl) contains need-1
      if ((long long)excl < need && need <= (long long)incl) {
        unsigned c = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((long long)(c + v[j]) >= need) {
            sm.digit = lane * 8 + j;
            sm.need = need - c;
            sm.cnt = v[j];
            break;
          }
          c += v[j];
        }
      }
    }
    __syncthreads();
    need = sm.need;
    prefix = (prefix << width) | (uint64_t)sm.digit;
    pshift = shift;
    const bool fin = (shift == 0) || (!value_mode && (long long)sm.cnt == need) || --max_passes == 0;
    __syncthreads();
    if (fin) break;
    shift = shift - 8 > 0 ? shift - 8 : 0;
  }
  *pshift_out = pshift;
  return prefix;
}

template <int NT, typename LoadF>
__device__ uint64_t cta_select_upper(int64_t n, int64_t kth, LoadF load, int passes, SelectSmem& sm) {
  int ps = 0;
  const uint64_t pre = cta_select<NT>(n, kth, load, true, &ps, sm, passes);
  return ps == 0 ? pre : ((pre << ps) | ((1ull << ps) - 1ull));
}

}  // namespace bbc
