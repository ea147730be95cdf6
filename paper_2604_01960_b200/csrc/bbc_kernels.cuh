// Kernels of the BBC query hot path (sm_100a).  Steps a1..a8 of DESIGN.md section 1.
//
// Canonical arithmetic: every value that decides an integer (probe order,
// LUT entries, estimates, bucket ids) is computed with explicitly rounded intrinsics
// (__fadd_rn/__fsub_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn) in a fixed order, so no FMA contraction
// can change a rounding; the CPU oracle evaluates the same expression tree.
#pragma once
#include "bbc_device.cuh"
#include <type_traits>

namespace bbc {

// Per-micro-batch pointers (device), all per-query arrays indexed by the query's slot in the
// micro-batch.
struct Batch {
  int nq;             // queries in this micro-batch
  int nbuckets;       // B regular equal-width buckets over [d_min, d_max] (1..255; 255 = overflow)
  int nprobe;
  int k;
  long long budget;
  long long cap;      // per-query element capacity (sum of the nprobe largest local lists)
  const float* Q;     // [nq x d]
  float* coarse;      // [nq x nlist]        coarse d^2 scratch
  int* probe;         // [nq x nprobe]
  float* rq2;         // [nq x nprobe]
  int* poff;          // [nq x (nprobe+1)]   element offset of each probed list (local)
  int* popad;         // [nq x (nprobe+1)]   same with every list rounded up to 32 objects
  long long* rbase;   // [nq x nprobe]       loff[probe[j]] - poff[j]: row of element i = rbase[j] + i
  int* nsamp;         // [nq]                sample lists s (0 = tau infinity)
  float* edges;       // [nq x 2]            (d_min, d_max)
  int* hist;          // [nq x 256]
  int* tau;           // [nq]
  int* ncand;         // [nq]
  float* table;       // PQ LUT [nq x M x 256] | RaBitQ u [nq x D]
  uint8_t* cells;     // [nq x cap]
  int* cpos;          // [nq x cap]  candidate rows (list-ordered index of this shard)
  int* cid;           // [nq x cap]  candidate original ids
  float* val;         // [nq x cap]  sample estimates, then exact d^2 of candidates
  long long* stats;   // [5] sum n_o, sum |S*|, sum sample objects, shortlisted lists, sum
                      //     objects estimated by the PQ sample pass (k_sample_cells)
  const int* qperm;   // [nq] locality order of the queries (k_qperm): CTA row y -> query qperm[y]
  int2* items;        // [nq x rqg] scan work items (query, pass) of the current pass (k_scan_plan)
  long long* ostage2_ids;  // second output staging buffer (host path, double-buffered copies)
  float* ostage2_d2;
  int* nitems;        // [1] number of work items
  int* chunk;         // [nq x nchunk]  per-chunk candidate counts -> offsets (compaction)
  int* chunkj;        // [nq x nchunk]  probed list holding each chunk's first element
  int* sstart;        // [nq x nprobe]  first candidate of each (query, probe) pair (pairs with poff < n)
  uint8_t* rmap;      // [nq x 256]     equal-depth remap of the cells (remap_m > 0)
  int remap_m;        // 0: buckets are the equal-width cells; else m equal-depth buckets (R6)
  int4* rseg;         // [nq x (nprobe + cap/64)] re-rank pieces (query, first, length) in list order
  int* rs_cnt;        // [nlist + 1]    piece counts (rs_off[nlist] = #pieces)
  int* rs_off;        // [nlist + 1]
  int* rs_cur;        // [nlist + 1]
  // sweep order of the 8-bit PQ scan (k_sweep_order / k_item_*): probe positions sorted by list
  // id within the sample and the main segment, their padded prefix offsets, and the work items
  // sorted by the list holding their first object
  int* sperm;         // [nq x nprobe]      sorted position -> probe position
  int* spad;          // [nq x (nprobe+1)]  padded offsets in sorted order (spad[ns] = popad[ns])
  int2* items_s;      // [as items]         items in sweep order
  int* ikey;          // [as items]         first list of each item
  int* icnt;          // [nlist + 1]        items per first list -> offsets
  int* nest;          // [nq]  lists the PQ sample pass estimates (>= nsamp; == nsamp unless 8-bit
                      //       PQ: then the same array only when nest_item == 0)
  int nest_item;      // objects per sample-pass work item (8-bit PQ), 0: nest = nsamp
  // Algorithm 3 (bbc_alg3.cuh; allocated only when the bound-aware re-rank is on)
  uint16_t* a3lb;     // [nq x cap]  (a_lb | a_ub << 8) per probe-order position
  uint16_t* a3lc;     // [nq x cap]  the same per candidate slot
  int* a3ordu;        // [nq x cap]  B_u's candidate slots grouped by a_ub
  int* a3nall;        // [nq]        nprobe (the estimate pass covers every probed list)
  int* a3pos;         // [nq x cap]  probe-order position of each candidate (k_emit, list mode)
  int* a3tau;         // [nq]        Algorithm 3's tau (b.tau holds the compaction's bound)
  // Algorithm 4 (early re-ranking of IVF+PQ, bbc_set_early_rerank; allocated only when it is on)
  int* tpred;         // [nq]        predicted threshold bucket tau_pred
  float* early;       // [nq x cap]  exact d^2 the main scan pass computed, per probe-order position
};

// Index arrays on the device.
struct Dev {
  int kind, d, nlist, M, D, raw_u8;
  int ksub;                      // PQ centroids per sub-quantizer: 256 (8-bit) or 16 (4-bit)
  int metric;                    // BBC_METRIC_L2 | BBC_METRIC_IP (keys -<q, x>)
  long long n_local;
  const float* centroids;        // [nlist x d]
  const long long* loff;         // [nlist + 1] local list offsets (rows of this shard)
  const int* gsize;              // [nlist] global list sizes (all shards)
  const long long* ids;          // [n_local]
  const float* books;            // [M x 256 x dsub]
  const uint8_t* codes;          // [n_local x M]
  const float* P;                // [D x D]
  const float* wL;               // [nlist x D]
  const uint8_t* bits;           // [n_local x D/8]
  const float* factors;          // [n_local x 2]
  const void* raw;               // [n_local x d] f32 | u8
  // tensor-core probe (bbc_probe_tc.cuh): centroid mean, |c - mu|^2, max |c - mu|
  const float* cmu;              // [d]
  const float* cnorm;            // [nlist]
  float cmax;
  int probe_tc;                  // 1: coarse holds d~ (shortlist mode of k_probe_select)
  long long ct_bytes;            // bytes of the group-major code copy (bounds checks)
};

// ------------------------------------------------------------------------------------------
// a1  coarse probe: canonical d^2 of every (query, centroid), 64 x 64 tiles, 4 x 4 per thread.
// ------------------------------------------------------------------------------------------
constexpr int kPT = 64, kPK = 16;
template <bool IP>
__global__ void __launch_bounds__(256) k_probe_d2(const float* __restrict__ Q,
                                                  const float* __restrict__ C, float* __restrict__ out,
                                                  int nq, int nlist, int d) {
  __shared__ float sQ[kPK][kPT + 1];
  __shared__ float sC[kPK][kPT + 1];
  const int q0 = blockIdx.y * kPT, c0 = blockIdx.x * kPT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int t0 = 0; t0 < d; t0 += kPK) {
    for (int e = threadIdx.x; e < kPT * kPK; e += 256) {
      int r = e / kPK, t = e % kPK;
      int qq = q0 + r, cc = c0 + r, tt = t0 + t;
      sQ[t][r] = (qq < nq && tt < d) ? Q[(size_t)qq * d + tt] : 0.f;
      sC[t][r] = (cc < nlist && tt < d) ? C[(size_t)cc * d + tt] : 0.f;
    }
    __syncthreads();
    const int tmax = min(kPK, d - t0);
    for (int t = 0; t < tmax; ++t) {
      float qv[4], cv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = sQ[t][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) cv[j] = sC[t][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (IP) {                                    // inner product: acc += q_t c_t
            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(qv[i], cv[j]));
          } else {
            float df = __fsub_rn(qv[i], cv[j]);
            acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(df, df));
          }
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int qq = q0 + ty * 4 + i;
    if (qq >= nq) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int cc = c0 + tx + 16 * j;
      if (cc < nlist) out[(size_t)qq * nlist + cc] = IP ? -acc[i][j] : acc[i][j];
    }
  }
}

// Per query: the nprobe smallest (d^2, list) keys, sorted; list offsets and the sample rule.
//
// ix.probe_tc == 0: coarse holds the canonical d^2 (k_probe_d2): radix select + sort.
// ix.probe_tc == 1: coarse holds the tensor-core estimate d~ (k_probe_mma) with |d~ - d^2| <=
//   E(q); the shortlist {d~ <= T~ + 2E} (T~ = nprobe-th smallest d~) provably holds the
//   nprobe nearest lists (bbc_probe_tc.cuh); it is re-scored with the canonical d^2 and
//   sorted, so the probe lists equal the SIMT path's.  A shortlist longer than kMaxShort falls
//   back to canonical d^2 for every list.
constexpr int kSelNT = 1024;
#ifndef BBC_PROBE_PASSES
#define BBC_PROBE_PASSES 2                  // digit passes of the probe shortlist's threshold
#endif
constexpr int kMaxProbe = 2048;
constexpr int kMaxShort = 4096;
constexpr int kMaxDimTc = 1024;

__device__ __forceinline__ float canonical_d2(const float* sq, const float* __restrict__ c, int d) {
  float acc = 0.f;
  if ((d & 3) == 0) {                                // 16-byte loads, 8 in flight per thread
    const float4* c4 = reinterpret_cast<const float4*>(c);
    const float4* q4 = reinterpret_cast<const float4*>(sq);
    for (int t0 = 0; t0 < d / 4; t0 += 8) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < d / 4) x[u] = __ldg(c4 + t0 + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (t0 + u < d / 4) {
          const float4 qv = q4[t0 + u];
          float df = __fsub_rn(qv.x, x[u].x); acc = __fadd_rn(acc, __fmul_rn(df, df));
          df = __fsub_rn(qv.y, x[u].y); acc = __fadd_rn(acc, __fmul_rn(df, df));
          df = __fsub_rn(qv.z, x[u].z); acc = __fadd_rn(acc, __fmul_rn(df, df));
          df = __fsub_rn(qv.w, x[u].w); acc = __fadd_rn(acc, __fmul_rn(df, df));
        }
      }
    }
    return acc;
  }
  for (int t = 0; t < d; ++t) {
    const float df = __fsub_rn(sq[t], c[t]);
    acc = __fadd_rn(acc, __fmul_rn(df, df));
  }
  return acc;
}

__device__ __forceinline__ void bitonic_sort_keys(uint64_t* keys, int P2) {
  if (P2 <= kSelNT) {
    // one key per thread: exchanges at stride < 32 by warp shuffles (no barrier), larger
    // strides through shared memory
    const int t = threadIdx.x;
    uint64_t v = t < P2 ? keys[t] : ~0ull;
    for (int size = 2; size <= P2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        uint64_t o;
        if (stride >= 32) {
          __syncthreads();
          if (t < P2) keys[t] = v;
          __syncthreads();
          o = t < P2 ? keys[t ^ stride] : ~0ull;
        } else {
          o = __shfl_xor_sync(0xffffffffu, v, stride);
        }
        const bool keepmin = ((t & stride) == 0) == ((t & size) == 0);
        v = keepmin ? (o < v ? o : v) : (o > v ? o : v);
      }
    }
    __syncthreads();
    if (t < P2) keys[t] = v;
    __syncthreads();
    return;
  }
  if (P2 == 2 * kSelNT) {
    // two adjacent keys per thread (elements 2t, 2t + 1): stride 1 inside the thread, strides
    // 2..32 by shuffles with thread t ^ (stride / 2), larger strides through shared memory
    const int t = threadIdx.x;
    __syncthreads();
    uint64_t v0 = keys[2 * t], v1 = keys[2 * t + 1];
    for (int size = 2; size <= P2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const bool up = ((2 * t) & size) == 0;
        if (stride == 1) {
          const uint64_t lo = v0 < v1 ? v0 : v1, hi = v0 < v1 ? v1 : v0;
          v0 = up ? lo : hi;
          v1 = up ? hi : lo;
          continue;
        }
        const int h = stride >> 1;                    // partner thread distance
        uint64_t o0, o1;
        if (h >= 32) {
          __syncthreads();
          keys[2 * t] = v0;
          keys[2 * t + 1] = v1;
          __syncthreads();
          o0 = keys[2 * (t ^ h)];
          o1 = keys[2 * (t ^ h) + 1];
        } else {
          o0 = __shfl_xor_sync(0xffffffffu, v0, h);
          o1 = __shfl_xor_sync(0xffffffffu, v1, h);
        }
        const bool keepmin = (((2 * t) & stride) == 0) == up;
        v0 = keepmin ? (o0 < v0 ? o0 : v0) : (o0 > v0 ? o0 : v0);
        v1 = keepmin ? (o1 < v1 ? o1 : v1) : (o1 > v1 ? o1 : v1);
      }
    }
    __syncthreads();
    keys[2 * t] = v0;
    keys[2 * t + 1] = v1;
    __syncthreads();
    return;
  }
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P2 / 2; i += kSelNT) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const uint64_t a = keys[lo], c = keys[hi];
        if ((a > c) == up) { keys[lo] = c; keys[hi] = a; }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSelNT) k_probe_select(Batch b, Dev ix) {
  __shared__ SelectSmem sm;
  __shared__ uint64_t keys[kMaxShort];
  __shared__ __align__(16) float s_q[kMaxDimTc];
  __shared__ int s_count;
  __shared__ float s_red[kSelNT / 32];
  const int q = blockIdx.x;
  const int nlist = ix.nlist, nprobe = b.nprobe, d = ix.d;
  float* d2 = b.coarse + (size_t)q * nlist;
  auto load = [&](int64_t i) -> uint64_t {
    return ((uint64_t)f2key(d2[i]) << 32) | (uint32_t)i;
  };
  bool sorted = false;
  if (ix.probe_tc) {
    // |q - mu|^2 (any order: only the error bound uses it)
    float part = 0.f;
    for (int t = threadIdx.x; t < d; t += kSelNT) {
      const float x = b.Q[(size_t)q * d + t];
      s_q[t] = x;
      const float y = x - ix.cmu[t];
      part = fmaf(y, y, part);
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = part;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    float qn = 0.f;
    for (int w = 0; w < kSelNT / 32; ++w) qn += s_red[w];
    qn *= 1.0f + 0x1p-10f;                          // margin for this sum's own rounding
    const float E = 0x1p-12f * sqrtf(qn) * ix.cmax + 0x1p-11f * (qn + ix.cmax * ix.cmax);
    auto load32 = [&](int64_t i) -> uint64_t { return (uint64_t)f2key(d2[i]); };
    // T~ is only needed as a lower end of the shortlist threshold: an upper bound of the
    // nprobe-th smallest d~ from two 8-bit digit passes instead of the full selection keeps
    // every true top-nprobe list in the shortlist (a few more lists are re-scored)
    const float T = key2f((uint32_t)cta_select_upper<kSelNT>(nlist, nprobe, load32, BBC_PROBE_PASSES, sm));
    float thr = T + 2.0f * E;
    thr = thr + fabsf(thr) * 0x1p-20f + 0x1p-100f;  // round the threshold up
    for (int i = threadIdx.x; i < nlist; i += kSelNT)
      if (d2[i] <= thr) {
        const int at = atomicAdd(&s_count, 1);
        if (at < kMaxShort) keys[at] = (uint64_t)i;
      }
    __syncthreads();
    const int cnt = s_count;
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)&b.stats[3], (unsigned long long)cnt);
    if (cnt <= kMaxShort) {
      int P2 = 1;
      while (P2 < cnt) P2 <<= 1;
      for (int i = threadIdx.x; i < P2; i += kSelNT) {
        if (i < cnt) {
          const int j = (int)keys[i];
          const float e = canonical_d2(s_q, ix.centroids + (size_t)j * d, d);
          keys[i] = ((uint64_t)f2key(e) << 32) | (uint32_t)j;
        } else {
          keys[i] = ~0ull;
        }
      }
      __syncthreads();
      bitonic_sort_keys(keys, P2);
      sorted = true;
    } else {
      for (int i = threadIdx.x; i < nlist; i += kSelNT)   // fallback: canonical d^2 everywhere
        d2[i] = canonical_d2(s_q, ix.centroids + (size_t)i * d, d);
      __syncthreads();
    }
  }
  if (!sorted) {
    int pshift;
    uint64_t pref = cta_select<kSelNT>(nlist, nprobe, load, false, &pshift, sm);
    if (threadIdx.x == 0) s_count = 0;
    int P2 = 1;
    while (P2 < nprobe) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += kSelNT) keys[i] = ~0ull;
    __syncthreads();
    for (int i = threadIdx.x; i < nlist; i += kSelNT) {
      uint64_t k = load(i);
      if (shr64(k, pshift) <= pref) keys[atomicAdd(&s_count, 1)] = k;
    }
    __syncthreads();
    bitonic_sort_keys(keys, P2);
  }
  // write probes; prefix over local and global sizes
  int* pr = b.probe + (size_t)q * nprobe;
  float* rq = b.rq2 + (size_t)q * nprobe;
  int* po = b.poff + (size_t)q * (nprobe + 1);
  int* pp = b.popad + (size_t)q * (nprobe + 1);
  long long lrun = 0, grun = 0, prun = 0;
  int s = -1;
  for (int base = 0; base < nprobe; base += kSelNT) {
    const int j = base + threadIdx.x;
    int lsz = 0, gsz = 0;
    if (j < nprobe) {
      uint64_t k = keys[j];
      int L = (int)(k & 0xffffffffu);
      pr[j] = L;
      rq[j] = key2f((uint32_t)(k >> 32));
      lsz = (int)(ix.loff[L + 1] - ix.loff[L]);
      gsz = ix.gsize[L];
    }
    // inclusive scans of lsz and gsz across the block (two ranks via block_rank is not enough:
    // use warp scans + smem)
    __shared__ long long wl[kSelNT / 32], wg[kSelNT / 32], wpd[kSelNT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long il = lsz, ig = gsz, ipd = (lsz + 31) & ~31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long tl = __shfl_up_sync(0xffffffffu, il, o);
      long long tg = __shfl_up_sync(0xffffffffu, ig, o);
      long long tp = __shfl_up_sync(0xffffffffu, ipd, o);
      if (lane >= o) { il += tl; ig += tg; ipd += tp; }
    }
    if (lane == 31) { wl[wid] = il; wg[wid] = ig; wpd[wid] = ipd; }
    __syncthreads();
    if (wid == 0) {
      long long vl = wl[lane], vg = wg[lane], vp = wpd[lane];
      long long sl = vl, sg = vg, sp = vp;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long tl = __shfl_up_sync(0xffffffffu, sl, o);
        long long tg = __shfl_up_sync(0xffffffffu, sg, o);
        long long tp = __shfl_up_sync(0xffffffffu, sp, o);
        if (lane >= o) { sl += tl; sg += tg; sp += tp; }
      }
      wl[lane] = sl - vl;
      wg[lane] = sg - vg;
      wpd[lane] = sp - vp;
    }
    __syncthreads();
    const long long excl_l = lrun + wl[wid] + il - lsz;
    const long long incl_g = grun + wg[wid] + ig;
    if (j < nprobe) {
      po[j] = (int)excl_l;
      b.rbase[(size_t)q * nprobe + j] = ix.loff[pr[j]] - excl_l;
      pp[j] = (int)(prun + wpd[wid] + ipd - ((lsz + 31) & ~31));
    }
    // sample rule: first j with cumulative global size >= budget
    int cand = (j < nprobe && incl_g >= b.budget && incl_g - gsz < b.budget) ? j : -1;
    __shared__ int s_first;
    if (threadIdx.x == 0) s_first = -1;
    __syncthreads();
    if (cand >= 0) s_first = cand;
    __syncthreads();
    if (s < 0 && s_first >= 0) s = s_first;
    // block totals
    __shared__ long long tot_l, tot_g, tot_p;
    if (threadIdx.x == kSelNT - 1) { tot_l = wl[wid] + il; tot_g = wg[wid] + ig; tot_p = wpd[wid] + ipd; }
    __syncthreads();
    lrun += tot_l;
    grun += tot_g;
    prun += tot_p;
    __syncthreads();
  }
  __shared__ int s_ns;
  if (threadIdx.x == 0) {
    po[nprobe] = (int)lrun;
    pp[nprobe] = (int)prun;
    int ns;
    if (grun <= b.budget) ns = 0;
    else {
      int s0 = nprobe < kSampleMinLists ? nprobe : kSampleMinLists;
      ns = s + 1 > s0 ? s + 1 : s0;
    }
    b.nsamp[q] = ns;
    s_ns = ns;
  }
  if (b.nest != b.nsamp) {
    // lists estimated by the 8-bit PQ scan's sample pass (nest >= ns): the sample's last work
    // item (nest_item objects) is filled up with the whole lists that follow it in probe order,
    // whose bucket ids k_sample_cells then forms from the stored estimates, so the main pass
    // starts after them instead of scanning them in a partly filled item of its own.  The edges
    // come from the first ns lists only (k_select_edges): no result changes.
    __shared__ int s_more;
    if (threadIdx.x == 0) s_more = 0;
    __syncthreads();
    const int ns = s_ns;
    if (ns > 0) {
      const int target = (pp[ns] + b.nest_item - 1) / b.nest_item * b.nest_item;
      int more = 0;                                  // lists after the sample ending by target
      for (int j = ns + threadIdx.x; j < nprobe; j += kSelNT) more += pp[j + 1] <= target;
      if (more) atomicAdd(&s_more, more);
    }
    __syncthreads();
    if (threadIdx.x == 0) b.nest[q] = ns + s_more;
  }
}

// Locality order of the micro-batch's queries: sorted by (region of the nearest list, nearest
// list, query), region = nearest of 256 pivot centroids (ivf_load).  Queries of one region
// probe mostly the same lists, so scheduling their scan / re-rank CTAs together turns some
// repeated code and row reads into L2 hits.  Only the order of CTAs changes, never a result.
// One CTA, bitonic sort of (lrank[probe[q][0]] << 32 | q).
constexpr int kQpermMax = 1 << 14;          // 128 KB of keys
__global__ void __launch_bounds__(1024) k_qperm(Batch b, const int* lrank, int* perm) {
  extern __shared__ unsigned long long qk[];
  int P2 = 1;
  while (P2 < b.nq) P2 <<= 1;
  for (int i = threadIdx.x; i < P2; i += 1024)
    qk[i] = i < b.nq ? ((unsigned long long)lrank[b.probe[(size_t)i * b.nprobe]] << 32) | (unsigned)i : ~0ull;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P2 / 2; i += 1024) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = qk[lo], c = qk[hi];
        if ((a > c) == up) { qk[lo] = c; qk[hi] = a; }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < b.nq; i += 1024) perm[i] = (int)(qk[i] & 0xffffffffu);
}

// ------------------------------------------------------------------------------------------
// a2  PQ lookup table: LUT[q][m][c] = sum_t (q_t - C[m][c][t])^2, t ascending (canonical)
// ------------------------------------------------------------------------------------------
// One CTA of ksub threads per (m, q); entry (m, c) at b.table[q * M * 256 + m * ksub + c].
__global__ void __launch_bounds__(256) k_pq_lut(Batch b, Dev ix) {
  const int m = blockIdx.x, q = blockIdx.y, c = threadIdx.x;
  const int ds = ix.d / ix.M;
  const float* qv = b.Q + (size_t)q * ix.d + m * ds;
  const float* cb = ix.books + ((size_t)m * ix.ksub + c) * ds;
  float acc = 0.f;
  if (ix.metric == BBC_METRIC_IP) {                   // LUT[m][c] = -<q_m, C[m][c]>
    for (int t = 0; t < ds; ++t) acc = __fadd_rn(acc, __fmul_rn(qv[t], cb[t]));
    acc = -acc;
  } else {
    for (int t = 0; t < ds; ++t) {
      float df = __fsub_rn(qv[t], cb[t]);
      acc = __fadd_rn(acc, __fmul_rn(df, df));
    }
  }
  b.table[(size_t)q * ix.M * 256 + (size_t)m * ix.ksub + c] = acc;
}

// RaBitQ rotated query u = P^T q: u_i = sum_{t<d} P[t][i] q_t, t ascending (canonical).
// CTA = (kRotNT output dims, QB queries): each P element is read once for QB queries (P is
// re-read nq / QB times from L2 instead of nq times), QB independent sums per thread.
constexpr int kRotNT = 128;   // output dims per CTA (1000 queries, D = 960: 1000 CTAs)
template <int QB>
__global__ void __launch_bounds__(kRotNT) k_rbq_rotate(Batch b, Dev ix) {
  extern __shared__ __align__(16) float sq[];   // [d][QB]
  const int q0 = blockIdx.y * QB, i = blockIdx.x * kRotNT + threadIdx.x;
  for (int e = threadIdx.x; e < ix.d * QB; e += kRotNT) {
    const int t = e / QB, k = e % QB;
    sq[e] = q0 + k < b.nq ? b.Q[(size_t)(q0 + k) * ix.d + t] : 0.f;
  }
  __syncthreads();
  if (i >= ix.D) return;
  float acc[QB];
#pragma unroll
  for (int k = 0; k < QB; ++k) acc[k] = 0.f;
  // P column i in blocks of 16 rows, the next block's loads issued before this block's sums
  constexpr int kB = 16;
  const float* Pi = ix.P + i;
  const int nfull = ix.d / kB;
  float pc[kB], pn[kB];
#pragma unroll
  for (int u = 0; u < kB; ++u) pc[u] = nfull > 0 ? __ldg(Pi + (size_t)u * ix.D) : 0.f;
  for (int blk = 0; blk < nfull; ++blk) {
    const int t0 = blk * kB;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      pn[u] = blk + 1 < nfull ? __ldg(Pi + (size_t)(t0 + kB + u) * ix.D) : 0.f;
#pragma unroll
    for (int u = 0; u < kB; ++u)
#pragma unroll
      for (int k = 0; k < QB; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(pc[u], sq[(t0 + u) * QB + k]));
#pragma unroll
    for (int u = 0; u < kB; ++u) pc[u] = pn[u];
  }
  for (int t = nfull * kB; t < ix.d; ++t) {
    const float p = __ldg(Pi + (size_t)t * ix.D);
#pragma unroll
    for (int k = 0; k < QB; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(p, sq[t * QB + k]));
  }
#pragma unroll
  for (int k = 0; k < QB; ++k)
    if (q0 + k < b.nq) b.table[(size_t)(q0 + k) * ix.D + i] = acc[k];
}

// ------------------------------------------------------------------------------------------
// bucket id (Eq. 6 with DESIGN R3): precomputed per query
// ------------------------------------------------------------------------------------------
struct CellFn {
  float dmin, dmax, inv, bmax;  // bmax = B - 1
  bool degen;
  __device__ __forceinline__ void init(float lo, float hi, int nb) {
    dmin = lo;
    dmax = hi;
    bmax = (float)(nb - 1);
    float w = __fsub_rn(hi, lo);
    degen = !(w > 0.f);
    inv = degen ? 0.f : __fdiv_rn((float)nb, w);
    if (!degen && isinf(inv)) degen = true;
  }
  // branch-free: clamp(floor((x - dmin) * inv), 0, bmax); 0 if degenerate; 255 beyond dmax.
  // clamp(floor(f), 0, bmax) = floor(clamp(f, 0, bmax)) (integer bounds; NaN -> 0), and floor of
  // y in [0, 255] is the low byte of fl_down(y + 2^23): no conversion-pipe instructions.
  __device__ __forceinline__ int operator()(float x) const {
    const float y = fminf(fmaxf(__fmul_rn(__fsub_rn(x, dmin), inv), 0.f), bmax);
    int c = __float_as_int(__fadd_rd(y, 8388608.0f)) & 0xFF;
    c = degen ? 0 : c;
    return x > dmax ? 255 : c;
  }
};

constexpr int kScanNT = 256;   // RaBitQ scan CTA size

// ------------------------------------------------------------------------------------------
// a3/a4  PQ code scan with a replicated LUT (query-major, conflict-free).
//
// CTA = (query q, pass P): objects [P*kRqE, (P+1)*kRqE) of q's probed objects in probe order,
// where every probed list starts on a multiple of 32 (padded order, popad), so a 32-object
// group never straddles two lists.  Warp w owns groups [32w, 32w + 32); lane l handles objects
// 4(l&7) .. 4(l&7)+3 of groups 32w + (l>>3) + 4i, i = 0..7 (32 objects, 32 running estimates
// in registers across all chunks).  The M sub-quantizers are visited in chunks of 4
// (canonical order m = 0..M-1); a lane fetches the 4 objects' code words of one group and chunk
// with one 16-byte load (8 lanes cover the group's 128 bytes: coalesced).
//
// The chunk's 4 x 256 LUT entries are replicated 32 times in shared memory so that lane l
// always reads bank l, whatever the code and whatever object it handles: no bank conflicts (a
// single LUT copy costs ~3.5 wavefronts per lookup with random codes).  The replica layout
// [mm>>1][c][mm&1][lane] makes the byte address of entry (mm, c) for lane l equal
// (c << 8) | 4l plus an immediate, so one byte permute of the code word gives the address:
// PRMT + LDS + FADD per lookup.  Group code offsets live in registers (no per-group pointer
// reads), and the first code loads of chunk p+1 are issued before the chunk barrier so the L2
// latency overlaps the LUT staging.
//   EST : estimate written to out_est[q * est_stride + probe-order position] (sample/debug)
//   !EST: bucket id to cells, histogram of ids < 255 (Push, Alg. 1 l.1-4)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

#ifndef BBC_RQ_WARPS
#define BBC_RQ_WARPS 32
#endif
#ifndef BBC_RQ_GPL
#define BBC_RQ_GPL 8
#endif
#ifndef BBC_RQ_DEPTH
#define BBC_RQ_DEPTH 2
#endif
constexpr int kRqWarps = BBC_RQ_WARPS, kRqNT = kRqWarps * 32;
constexpr int kRqGPL = BBC_RQ_GPL;                       // groups per lane (8)
constexpr int kRqEW = 4 * kRqGPL;                        // objects (running sums) per lane (32)
constexpr int kRqE = kRqNT * kRqEW;                      // objects per CTA work item (32768)
constexpr int kRqMC = 4;                                 // sub-quantizers per chunk
constexpr int kRqDepth = BBC_RQ_DEPTH;                   // 16-byte code loads in flight per lane
constexpr int kRqGroups = kRqWarps * 4 * kRqGPL;         // 32-object groups per CTA
constexpr int kRqLutBytes = kRqMC * 256 * 32 * 4;        // 131072
// dynamic shared memory: [LUT chunk][group code offsets][group output offsets][group counts]
//                        [histogram][padded probe offsets]
constexpr int kRqOffGo = kRqLutBytes;
constexpr int kRqOffOut = kRqOffGo + kRqGroups * 4;
constexpr int kRqOffCnt = kRqOffOut + kRqGroups * 8;
constexpr int kRqOffHist = kRqOffCnt + kRqGroups * 4;
constexpr int kRqOffPo = kRqOffHist + kCells * 4;
constexpr size_t kRqSmem = kRqOffPo + (kMaxProbe + 1) * 4;
// The kernel has no static shared memory, so its dynamic buffer starts right after the 1 KB
// the driver reserves per CTA; the LUT lookups use that offset as an immediate (checked).
constexpr unsigned kRqSmemBase = 1024;

// Codes in group-major order for this scan: list L is cut into groups of 32 objects; group g,
// chunk p (sub-quantizers 4p..4p+3), object lane l at byte tbase[L] + (g*(M/4) + p)*128 + 4l.
// Every list's byte size is a multiple of 128 (M % 4 == 0), so offsets are kept in 128-byte units.
__device__ __forceinline__ long long rq_list_bytes(int n, int M) { return (long long)((n + 31) >> 5) * M * 32; }
constexpr int kCodesTailPad = 128;

template <int IMM>
__device__ __forceinline__ float lds_imm(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(IMM));
  return v;
}

template <int N, typename F, int I = 0>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, F, I + 1>(static_cast<F&&>(f));
  }
}

// acc += the 4 LUT entries selected by code word w (sub-quantizers 4p..4p+3, canonical order)
__device__ __forceinline__ float rq_lookup4(float a, uint32_t w, uint32_t lane4) {
  a = __fadd_rn(a, lds_imm<kRqSmemBase + 0>(__byte_perm(w, lane4, 0x7604)));
  a = __fadd_rn(a, lds_imm<kRqSmemBase + 128>(__byte_perm(w, lane4, 0x7614)));
  a = __fadd_rn(a, lds_imm<kRqSmemBase + 65536>(__byte_perm(w, lane4, 0x7624)));
  a = __fadd_rn(a, lds_imm<kRqSmemBase + 65536 + 128>(__byte_perm(w, lane4, 0x7634)));
  return a;
}

// mode 0: sample lists [0, nsamp) -> estimates; 1: lists [nsamp, nprobe) -> bucket ids;
// 2: all lists -> estimates (debug)
// NOALLOC: code loads bypass L1 allocation (codes larger than L2 are streamed once from HBM:
// C4/C5 +1.5 %; L2-resident codes (C2) are faster through L1)
// Algorithm 4: the contribution of 16 row bytes (chunk t) to the exact key: sum (x - q)^2, or
// sum x q for the inner product; fp32 rows hold 4 values per chunk, uint8 rows 16.
__device__ __forceinline__ float early_part(float a, const uint4& x, const float* __restrict__ qv, int t,
                                            bool u8, bool ipm) {
  if (u8) {
    const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float4 y = __ldg(reinterpret_cast<const float4*>(qv) + 4 * t + h);
      const float ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int by = 0; by < 4; ++by) {
        const float xv = (float)((wv[h] >> (8 * by)) & 255u);
        if (ipm) a = fmaf(xv, ys[by], a);
        else { const float df = xv - ys[by]; a = fmaf(df, df, a); }
      }
    }
  } else {
    const float4 y = __ldg(reinterpret_cast<const float4*>(qv) + t);
    const float xs[4] = {__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z), __uint_as_float(x.w)};
    const float ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (ipm) a = fmaf(xs[h], ys[h], a);
      else { const float df = xs[h] - ys[h]; a = fmaf(df, df, a); }
    }
  }
  return a;
}

template <int M, bool EST, bool NOALLOC = false>
__global__ void __launch_bounds__(kRqNT, 1) k_pq_scan_rq(Batch b, Dev ix, const uint8_t* __restrict__ codes_t,
                                                         const long long* __restrict__ tbase,
                                                         float* out_est, long long est_stride,
                                                         int mode, const int2* __restrict__ items,
                                                         const int* __restrict__ nitems,
                                                         const int* __restrict__ sperm) {
  constexpr int P = M / kRqMC;                       // chunks
  extern __shared__ __align__(16) uint8_t rsm[];
  float* lut = reinterpret_cast<float*>(rsm);
  uint32_t* gofs = reinterpret_cast<uint32_t*>(rsm + kRqOffGo);
  long long* gout = reinterpret_cast<long long*>(rsm + kRqOffOut);
  int* gcnt = reinterpret_cast<int*>(rsm + kRqOffCnt);
  int* hist = reinterpret_cast<int*>(rsm + kRqOffHist);
  int* s_popad = reinterpret_cast<int*>(rsm + kRqOffPo);
  // persistent CTAs over the work items of k_scan_plan: (query, pass) in query locality order
  // (probe order) or sorted by their first list (sweep order)
  const int nit = *nitems;
  for (int it = blockIdx.x; it < nit; it += gridDim.x) {
  __syncthreads();                                   // shared memory of the previous item free
  const int2 wk = items[it];
  const int q = wk.x;
  BBC_CHECK(q >= 0 && q < b.nq && wk.y >= 0);
  const int ns = b.nest[q];                          // lists of the sample pass (>= nsamp)
  if (mode != 2 && ns == 0) continue;                // tau = infinity: nothing to bucket
  const int first = mode == 1 ? ns : 0;
  const int lim = mode == 0 ? ns : b.nprobe;
  // padded offsets in visiting order: probe order (sperm == null) or sweep order (k_sweep_order)
  const int* popad = (sperm ? b.spad : b.popad) + (size_t)q * (b.nprobe + 1);
  const int* sp = sperm ? sperm + (size_t)q * b.nprobe : nullptr;
  const int nflat = popad[lim];
  const int x0 = popad[first] + wk.y * kRqE;
  if (x0 >= nflat) continue;
  if (smem_u32(rsm) != kRqSmemBase) __trap();        // layout assumption of lds_imm
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = threadIdx.x; j <= lim; j += kRqNT) s_popad[j] = popad[j];
  if (!EST)
    for (int i = threadIdx.x; i < kCells; i += kRqNT) hist[i] = 0;
  const float* glut = b.table + (size_t)q * M * 256;
  constexpr int kStage = (kRqMC * 256 + kRqNT - 1) / kRqNT;   // LUT entries staged per thread
  float nv[kStage];
#pragma unroll
  for (int h = 0; h < kStage; ++h)
    nv[h] = threadIdx.x + h * kRqNT < kRqMC * 256 ? __ldg(glut + threadIdx.x + h * kRqNT) : 0.f;   // chunk 0
  __syncthreads();
  // group table: group G = 32 objects starting at flat x0 + 32 G (never straddles a list)
  const int* po = b.poff + (size_t)q * (b.nprobe + 1);
  const int* pr = b.probe + (size_t)q * b.nprobe;
  const long long obase = EST ? (long long)q * est_stride : (long long)q * b.cap;
  for (int G = threadIdx.x; G < kRqGroups; G += kRqNT) {
    uint32_t go = 0;                                  // invalid groups read (masked) list 0
    long long oo = 0;
    int cnt = 0;
    const int xg = x0 + 32 * G;
    if (xg < nflat) {
      int lo = first, hi = lim - 1;                   // last j with popad[j] <= xg
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_popad[mid] <= xg) lo = mid; else hi = mid - 1;
      }
      const int j = sp ? sp[lo] : lo;                // probe position of the group's list
      BBC_CHECK(lo >= first && lo < lim && j >= 0 && j < b.nprobe);
      const int L = pr[j];
      BBC_CHECK(L >= 0 && L < ix.nlist);
      const int nL = (int)(ix.loff[L + 1] - ix.loff[L]);
      const int i0 = xg - s_popad[lo];
      BBC_CHECK(i0 >= 0 && i0 < nL && (i0 & 31) == 0);
      cnt = min(32, nL - i0);
      go = (uint32_t)((tbase[L] + (long long)(i0 >> 5) * M * 32) >> 7);
      BBC_CHECK(((long long)go << 7) + (long long)M * 32 <= ix.ct_bytes);
      oo = obase + po[j] + i0;
      BBC_CHECK(po[j] + i0 + cnt <= (EST ? est_stride : b.cap));
    }
    gofs[G] = go;
    gout[G] = oo;
    gcnt[G] = cnt;
  }
  __syncthreads();
  const int gl0 = wid * 4 * kRqGPL + (lane >> 3);    // the lane's groups: gl0 + 4 i
  // 16-byte index of the lane's slice of group gl0 + 4i, chunk p: gofs*8 + (lane&7) + 8p.  The
  // group offsets are re-read from shared memory per load (4 distinct words per warp: one
  // wavefront per 16 lookups) rather than held in 8 registers, which would spill.
  for (int G = threadIdx.x; G < kRqGroups; G += kRqNT) gofs[G] = gofs[G] * 8u;
  __syncthreads();
  const uint32_t gaddr = smem_u32(gofs + gl0);
  const uint4* __restrict__ c16 = reinterpret_cast<const uint4*>(codes_t) + (lane & 7);
  auto ldc = [&](auto ic, int p) -> uint4 {
    uint32_t g;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(g) : "r"(gaddr), "n"(16 * decltype(ic)::value));
    if (NOALLOC) {
      uint4 r;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(c16 + (g + 8u * (uint32_t)p)));
      return r;
    }
    return __ldg(c16 + (g + 8u * (uint32_t)p));
  };
  float acc[kRqEW];
#pragma unroll
  for (int e = 0; e < kRqEW; ++e) acc[e] = 0.f;
  const uint32_t lane4 = (uint32_t)lane * 4u;
  // sample pass over L2-resident codes (EST, !NOALLOC): a warp whose groups all lie past the
  // item's objects (valid groups form a prefix; a query's sample ends in a partly filled item)
  // only stages and syncs (C2 sample 0.39 -> 0.35 ms).  Elsewhere the loop stays unconditional:
  // the branch measured slower on the main pass (C4 50.2 -> 54.2 ms) and on C4's streamed sample
  // pass (14.1 -> 14.8 ms).
  const bool wact = !(EST && !NOALLOC) || gcnt[wid * 4 * kRqGPL] > 0;
  uint4 cw[kRqDepth];
  if (wact) static_for<kRqDepth>([&](auto ic) { cw[decltype(ic)::value] = ldc(ic, 0); });
#pragma unroll 1
  for (int p = 0; p < P; ++p) {
    __syncthreads();                                  // previous chunk fully consumed
    // stage chunk p: entry (mm, c) replicated 32x at words ((mm>>1)*256 + c)*64 + (mm&1)*32 +
    // [0, 32): lane l reads bank l.  Each thread writes its entries as 8 rotated 16-byte
    // stores each (a quarter-warp covers all 32 banks).
#pragma unroll
    for (int h = 0; h < kStage; ++h) {
      const float4 a4 = make_float4(nv[h], nv[h], nv[h], nv[h]);
      const int ea = threadIdx.x + h * kRqNT;
      if ((kRqMC * 256) % kRqNT == 0 || ea < kRqMC * 256) {
        float4* ra = reinterpret_cast<float4*>(lut + (size_t)((ea >> 9) * 256 + (ea & 255)) * 64 + ((ea >> 8) & 1) * 32);
#pragma unroll
        for (int r = 0; r < 8; ++r) ra[(r + lane) & 7] = a4;
      }
    }
    if (p + 1 < P) {                                  // prefetch chunk p+1's entries
#pragma unroll
      for (int h = 0; h < kStage; ++h)
        if ((kRqMC * 256) % kRqNT == 0 || threadIdx.x + h * kRqNT < kRqMC * 256)
          nv[h] = __ldg(glut + (p + 1) * kRqMC * 256 + threadIdx.x + h * kRqNT);
    }
    __syncthreads();
    const int pn = p + 1 < P ? p + 1 : p;            // code loads run one chunk ahead at the tail
    if (wact) static_for<kRqGPL>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      const uint4 c = cw[i % kRqDepth];
      if constexpr (i + kRqDepth < kRqGPL)
        cw[i % kRqDepth] = ldc(std::integral_constant<int, i + kRqDepth>{}, p);
      else
        cw[i % kRqDepth] = ldc(std::integral_constant<int, i + kRqDepth - kRqGPL>{}, pn);
      acc[4 * i + 0] = rq_lookup4(acc[4 * i + 0], c.x, lane4);
      acc[4 * i + 1] = rq_lookup4(acc[4 * i + 1], c.y, lane4);
      acc[4 * i + 2] = rq_lookup4(acc[4 * i + 2], c.z, lane4);
      acc[4 * i + 3] = rq_lookup4(acc[4 * i + 3], c.w, lane4);
    });
  }
  // epilogue: lane l holds objects 4(l&7)+j of its groups
  CellFn cf;
  if (!EST) cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
#pragma unroll
  for (int i = 0; i < kRqGPL; ++i) {
    const int G = gl0 + 4 * i;
    const int cnt = gcnt[G];
    const long long oo = gout[G] + 4 * (lane & 7);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // plain per-lane shared atomics: warp aggregation (warp_hist_add) measured slower here
      // (C4 scan 73 -> 98 ms: ~89 % of the ids are the uncounted 255 and the rest spread over
      // 255 cells, so contention is low and the match costs more than it saves)
      if (4 * (lane & 7) + j < cnt) {
        if (EST) {
          out_est[oo + j] = acc[4 * i + j];
        } else {
          const int cell = cf(acc[4 * i + j]);
          b.cells[oo + j] = (uint8_t)cell;
          if (cell < 255) atomicAdd(&hist[cell], 1);
        }
      }
    }
  }
  if (!EST) {
    __syncthreads();
    for (int i = threadIdx.x; i < kCells; i += kRqNT)
      if (hist[i]) atomicAdd(&b.hist[(size_t)q * kCells + i], hist[i]);
  }
  }
}

// Work items of a scan pass: every (query, item_objs-object pass) that has objects, in query
// locality order (qperm), so the scan runs as persistent CTAs without idle blocks (a static
// grid sized for the largest query left most CTAs of small queries empty).  One CTA.
//   mode 0: sample lists [0, nsamp); 1: lists [nsamp, nprobe); 2: all lists.
__global__ void __launch_bounds__(1024) k_scan_plan(Batch b, int mode, int2* items, int* nitems, int item_objs) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < b.nq; base += 1024) {
    const int r = base + threadIdx.x;
    int cnt = 0, q = 0;
    if (r < b.nq) {
      q = b.qperm[r];
      const int ns = b.nest[q];
      if (mode == 2 || ns > 0) {
        const int* pp = b.popad + (size_t)q * (b.nprobe + 1);
        const int first = mode == 1 ? ns : 0, lim = mode == 0 ? ns : b.nprobe;
        cnt = (pp[lim] - pp[first] + item_objs - 1) / item_objs;
      }
    }
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int v = ws[lane];
      int y = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      ws[lane] = y - v;
    }
    __syncthreads();
    const int off = carry + ws[wid] + x - cnt;
    for (int c = 0; c < cnt; ++c) items[off + c] = make_int2(q, c);
    __syncthreads();
    if (threadIdx.x == 1023) carry = off + cnt;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nitems = carry;
}

// Sweep order of the 8-bit PQ scan (codes larger than L2).  In probe order the CTAs that run
// at the same time scan unrelated lists of unrelated queries, so every (query, list) pair pulls
// the list's codes from HBM again (C4: DRAM reads 0.76x the algorithmic code bytes).  In sweep
// order each query's lists are visited by ascending list id and the work items are issued by the
// list holding their first object: the ~148 items in flight then cover one window of the list-id
// space (C4: an item spans ~50 lists, ~1,100 list ids, ~33 MB of codes), which stays in L2 while
// the other queries' items that start in it pass.  Only the visiting order changes: every
// object's estimate / bucket id still goes to its probe-order position (poff), so the results are
// identical bit for bit.
//
// k_sweep_order: one CTA (kSelNT threads) per query.  Probe positions sorted by (segment, list
// id) -- segment 0 = the sample lists [0, ns), 1 = the rest -- and the padded prefix offsets in
// that order (the segment totals equal popad's: spad[ns] = popad[ns], spad[nprobe] = popad[nprobe]).
__global__ void __launch_bounds__(kSelNT) k_sweep_order(Batch b, Dev ix) {
  __shared__ uint64_t keys[kMaxProbe];
  __shared__ int ws[kSelNT / 32];
  __shared__ int carry;
  const int q = blockIdx.x, np = b.nprobe, ns = b.nest[q];
  const int* pr = b.probe + (size_t)q * np;
  int P2 = 1;
  while (P2 < np) P2 <<= 1;
  for (int i = threadIdx.x; i < P2; i += kSelNT)
    keys[i] = i < np ? ((uint64_t)(i >= ns) << 63) | ((uint64_t)pr[i] << 24) | (uint64_t)i : ~0ull;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  bitonic_sort_keys(keys, P2);
  __syncthreads();
  int* sp = b.sperm + (size_t)q * np;
  int* pd = b.spad + (size_t)q * (np + 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < np; base += kSelNT) {
    const int t = base + threadIdx.x;
    int sz = 0, j = 0;
    if (t < np) {
      j = (int)(keys[t] & 0xffffffu);
      BBC_CHECK(j < np && (t < ns) == (j < ns));
      const int L = pr[j];
      sz = ((int)(ix.loff[L + 1] - ix.loff[L]) + 31) & ~31;
      sp[t] = j;
    }
    int x = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int v = ws[lane];
      int y = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      ws[lane] = y - v;
    }
    __syncthreads();
    if (t < np) pd[t] = carry + ws[wid] + x - sz;
    __syncthreads();
    if (threadIdx.x == kSelNT - 1) carry += ws[wid] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) pd[np] = carry;
}

// Sweep-ordered work items: a counting sort of k_scan_plan's items by the list holding their
// first object.  k_item_count: that list per item (binary search of the item's first padded
// position in spad) and the per-list counts; k_item_offsets: exclusive scan of the counts (one
// CTA); k_item_scatter: items to their list's slots (order inside a list unspecified -- it changes
// no result: items write disjoint outputs and add integer counts).
__global__ void __launch_bounds__(256) k_item_count(Batch b, int mode, int item_objs, int ix_nlist) {
  const int nit = *b.nitems;
  for (int it = blockIdx.x * 256 + threadIdx.x; it < nit; it += gridDim.x * 256) {
    const int2 wk = b.items[it];
    const int q = wk.x, ns = b.nest[q];
    const int first = mode == 1 ? ns : 0, lim = mode == 0 ? ns : b.nprobe;
    const int* pd = b.spad + (size_t)q * (b.nprobe + 1);
    const int x = pd[first] + wk.y * item_objs;
    int lo = first, hi = lim - 1;                      // last t with spad[t] <= x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pd[mid] <= x) lo = mid; else hi = mid - 1;
    }
    const int L = b.probe[(size_t)q * b.nprobe + b.sperm[(size_t)q * b.nprobe + lo]];
    BBC_CHECK(lo >= first && lo < lim && L >= 0 && L < ix_nlist);
    b.ikey[it] = L;
    atomicAdd(&b.icnt[L], 1);
  }
}

__global__ void __launch_bounds__(1024) k_item_offsets(int* cnt, int n) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? cnt[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int w = ws[lane];
      int y = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      ws[lane] = y - w;
    }
    __syncthreads();
    if (i < n) cnt[i] = carry + ws[wid] + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += ws[wid] + x;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_item_scatter(Batch b) {
  const int nit = *b.nitems;
  for (int it = blockIdx.x * 256 + threadIdx.x; it < nit; it += gridDim.x * 256) {
    const int at = atomicAdd(&b.icnt[b.ikey[it]], 1);
    BBC_CHECK(at >= 0 && at < nit);
    b.items_s[at] = b.items[it];
  }
}

// Index-load-time copy of the PQ codes in the group-major order of k_pq_scan_rq.
__global__ void k_transpose_codes(const uint8_t* codes, const long long* loff,
                                  const long long* tbase, int nlist, long long n, int M,
                                  uint8_t* codes_t) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int lo = 0, hi = nlist - 1;                         // last list with loff[L] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (loff[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const int L = lo;
  const long long x = r - loff[L];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(codes + r * M);
  uint8_t* dst = codes_t + tbase[L] + (x >> 5) * M * 32 + (x & 31) * 4;
  for (int p = 0; p < M / 4; ++p) *reinterpret_cast<uint32_t*>(dst + p * 128) = src[p];
}

// Bucket ids (and histogram) of the sample objects from their stored estimates, once the edges
// are known (the list-major main scan skips the sample pairs).
__global__ void __launch_bounds__(256) k_sample_cells(Batch b) {
  __shared__ int hist[kCells];
  const int q = blockIdx.y;
  const int ns = b.nest[q];                          // the sample and its fill-up lists
  if (ns == 0) return;
  const int n = b.poff[(size_t)q * (b.nprobe + 1) + ns];
  BBC_CHECK(n <= b.cap);
  if (blockIdx.x == 0 && threadIdx.x == 0)          // objects estimated by the sample pass
    atomicAdd((unsigned long long*)&b.stats[4], (unsigned long long)n);
  if (blockIdx.x * 1024 >= n) return;
  for (int i = threadIdx.x; i < kCells; i += 256) hist[i] = 0;
  CellFn cf;
  cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
  __syncthreads();
  const float* v = b.val + (size_t)q * b.cap;
  uint8_t* cl = b.cells + (size_t)q * b.cap;
  // four consecutive estimates per thread and step: one 16-byte load, one 4-byte store of their
  // bucket ids (cap is a multiple of 16, so the query's rows are aligned); two steps in flight
  const int stride = gridDim.x * 256 * 4;
  for (int i0 = (blockIdx.x * 256 + threadIdx.x) * 4; i0 < n; i0 += 2 * stride) {
    float4 x[2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
      x[u] = i0 + u * stride < n ? *reinterpret_cast<const float4*>(v + i0 + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * stride;
      if (i >= n) break;
      const float e[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
      uint32_t w = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int c = i + t < n ? cf(e[t]) : 255;
        w |= (uint32_t)c << (8 * t);
        if (c < 255) atomicAdd(&hist[c], 1);
      }
      if (i + 4 <= n) *reinterpret_cast<uint32_t*>(cl + i) = w;
      else
        for (int t = 0; i + t < n; ++t) cl[i + t] = (uint8_t)(w >> (8 * t));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kCells; i += 256)
    if (hist[i]) atomicAdd(&b.hist[(size_t)q * kCells + i], hist[i]);
}

// ------------------------------------------------------------------------------------------
// a3/a4  RaBitQ scan: per (query, list) 4-bit query code as 4 bit planes in shared memory, then
// ip = <bits, qbar> = sum_p 2^p popc(bits & plane_p) per object (B_q = 4).
// ------------------------------------------------------------------------------------------
template <bool SAMPLE>
__global__ void __launch_bounds__(kScanNT) k_rbq_scan(Batch b, Dev ix, int G) {
  extern __shared__ float smem[];
  const int D = ix.D, W = D / 32;
  float* qp = smem;                                       // [D]
  uint32_t* planes = reinterpret_cast<uint32_t*>(smem + D); // [4 x W]
  __shared__ int hist[kCells];
  __shared__ float red_mn[kScanNT / 32], red_mx[kScanNT / 32];
  __shared__ int red_s[kScanNT / 32];
  __shared__ float s_c[4];
  const int q = blockIdx.y;
  const int ns = b.nsamp[q];
  if (ns == 0) return;
  const int jlim = SAMPLE ? ns : b.nprobe;
  if (blockIdx.x * G >= jlim) return;
  CellFn cf;
  if (!SAMPLE) {
    for (int i = threadIdx.x; i < kCells; i += kScanNT) hist[i] = 0;
    cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
  }
  const float* u = b.table + (size_t)q * D;
  const int* po = b.poff + (size_t)q * (b.nprobe + 1);
  const int* pr = b.probe + (size_t)q * b.nprobe;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int g0 = blockIdx.x * G; g0 < jlim; g0 += gridDim.x * G)
  for (int j = g0; j < min(g0 + G, jlim); ++j) {
    const int L = pr[j];
    const float rq2 = b.rq2[(size_t)q * b.nprobe + j];
    const float r = __fsqrt_rn(rq2);
    const float* w = ix.wL + (size_t)L * D;
    const float rinv = r > 0.f ? __fdiv_rn(1.0f, r) : 0.f;
    float mn = INFINITY, mx = -INFINITY;
    for (int i = threadIdx.x; i < D; i += kScanNT) {
      float v = r > 0.f ? __fmul_rn(__fsub_rn(u[i], w[i]), rinv) : 0.f;
      qp[i] = v;
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (lane == 0) { red_mn[wid] = mn; red_mx[wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float a = red_mn[0], c = red_mx[0];
      for (int t = 1; t < kScanNT / 32; ++t) { a = fminf(a, red_mn[t]); c = fmaxf(c, red_mx[t]); }
      s_c[0] = a;
      s_c[1] = __fdiv_rn(__fsub_rn(c, a), 15.0f);
    }
    __syncthreads();
    const float vl = s_c[0], delta = s_c[1];
    const float dinv = delta > 0.f ? __fdiv_rn(1.0f, delta) : 0.f;
    int sq = 0;
    for (int base = 0; base < D; base += kScanNT) {      // D is a multiple of 64
      const int i = base + threadIdx.x;
      int qb = 0;
      if (i < D && delta > 0.f) {
        float t = floorf(__fadd_rn(__fmul_rn(__fsub_rn(qp[i], vl), dinv), 0.5f));
        qb = t < 0.f ? 0 : (t > 15.f ? 15 : (int)t);
      }
      sq += qb;
      const bool act = (base + wid * 32) < D;
      if (act) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          unsigned m = __ballot_sync(0xffffffffu, (qb >> p) & 1);
          if (lane == 0) planes[p * W + (i >> 5)] = m;
        }
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) red_s[wid] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int t = 0; t < kScanNT / 32; ++t) s += red_s[t];
      const float sD = __fsqrt_rn((float)D);
      s_c[0] = __fdiv_rn(__fmul_rn(2.0f, delta), sD);                               // c1
      s_c[1] = __fdiv_rn(__fmul_rn(2.0f, vl), sD);                                  // c2
      s_c[2] = __fsub_rn(-__fdiv_rn(__fmul_rn(delta, (float)s), sD), __fmul_rn(sD, vl)); // c3
    }
    __syncthreads();
    const float c1 = s_c[0], c2 = s_c[1], c3 = s_c[2];
    const long long row0 = ix.loff[L];
    const int n = (int)(ix.loff[L + 1] - row0);
    const long long e0 = (long long)q * b.cap + po[j];
    for (int i0 = 0; i0 < n; i0 += kScanNT) {           // warp-uniform trip count (warp_hist_add)
      const int i = i0 + threadIdx.x;
      if (i >= n) {
        if (!SAMPLE) warp_hist_add(hist, 255);
        continue;
      }
      const uint2* bp = reinterpret_cast<const uint2*>(ix.bits + (size_t)(row0 + i) * (D / 8));
      int ip = 0, pc = 0;
      for (int v = 0; v < W / 2; ++v) {
        uint2 x = __ldg(bp + v);
        const int w0 = 2 * v;
        pc += __popc(x.x) + __popc(x.y);
#pragma unroll
        for (int p = 0; p < 4; ++p)
          ip += (__popc(x.x & planes[p * W + w0]) + __popc(x.y & planes[p * W + w0 + 1])) << p;
      }
      const float2 f = __ldg(reinterpret_cast<const float2*>(ix.factors) + row0 + i);
      const float t1 = __fmul_rn(c2, (float)pc);
      const float t2 = __fadd_rn(t1, c3);
      const float t3 = __fmul_rn(c1, (float)ip);
      const float oq = __fadd_rn(t3, t2);
      const float e = __fmul_rn(oq, __fdiv_rn(1.0f, f.y));
      const float a = __fmul_rn(f.x, f.x);
      const float s = __fadd_rn(a, rq2);
      const float ff = __fmul_rn(__fmul_rn(2.0f, f.x), r);
      const float est = __fsub_rn(s, __fmul_rn(ff, e));
      if (SAMPLE) {
        b.val[e0 + i] = est;
      } else {
        const int cell = cf(est);
        b.cells[e0 + i] = (uint8_t)cell;
        warp_hist_add(hist, cell);
      }
    }
    __syncthreads();
  }
  if (!SAMPLE) {
    int* gh = b.hist + (size_t)q * kCells;
    for (int i = threadIdx.x; i < kCells; i += kScanNT)
      if (hist[i]) atomicAdd(&gh[i], hist[i]);
  }
}

// CTA radix selection of the kth smallest of n 32-bit keys (duplicates allowed) with 11-bit
// digits over the bits where the keys differ (<= 3 histogram passes after one min/max pass).
// key(i) -> (key, valid).  Returns the kth smallest valid key and, in *take, how many of the
// elements equal to it belong to the k smallest (kth - #smaller).  Requires kth <= #valid.
// DB-bit digits (2^DB histogram bins, 2^DB / 1024 per thread in the scan)
template <int DB>
struct Kth32SmemT {
  unsigned hist[1 << DB];
  unsigned wsum[32];
  unsigned mn[32], mx[32];
  unsigned prefix, digit, need, dcount;
};
using Kth32Smem = Kth32SmemT<11>;

// *eq_out (optional): how many keys equal the returned kth key (its bin in the last pass)
template <typename KeyF, int DB = 11>
__device__ uint32_t cta_kth32(int n, unsigned kth, KeyF key, unsigned* take, Kth32SmemT<DB>& sm,
                              uint32_t* min_out = nullptr, unsigned* eq_out = nullptr) {
  constexpr int NT = kSelNT;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned mn = 0xffffffffu, mx = 0u;
  for (int i = threadIdx.x; i < n; i += NT) {
    bool ok;
    const uint32_t k = key(i, &ok);
    if (ok) { mn = min(mn, k); mx = max(mx, k); }
  }
  mn = warp_min(mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) { sm.mn[wid] = mn; sm.mx[wid] = mx; }
  __syncthreads();
  if (wid == 0) {
    unsigned a = sm.mn[lane], c = sm.mx[lane];
    a = warp_min(a);
    c = __reduce_max_sync(0xffffffffu, c);
    if (lane == 0) { sm.mn[0] = a; sm.mx[0] = c; }
  }
  __syncthreads();
  mn = sm.mn[0];
  mx = sm.mx[0];
  if (min_out) *min_out = mn;
  __syncthreads();
  if (mn == mx || kth <= 1) {
    if (mn == mx) {
      *take = kth;
      if (eq_out) *eq_out = (unsigned)n;             // (every key valid: the callers' case)
      return mn;
    }
  }
  int hi = 31 - __clz(mn ^ mx);                       // highest differing bit
  uint32_t prefix = hi == 31 ? 0u : (mn >> (hi + 1));
  int pshift = hi + 1;
  unsigned need = kth;
  while (true) {
    const int shift = max(0, pshift - DB);
    const int width = pshift - shift;
    const unsigned mask = (1u << width) - 1u;
    for (int i = threadIdx.x; i < (1 << DB); i += NT) sm.hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
      bool ok;
      const uint32_t k = key(i, &ok);
      if (ok && (pshift == 32 || (k >> pshift) == prefix)) atomicAdd(&sm.hist[(k >> shift) & mask], 1u);
    }
    __syncthreads();
    // exclusive scan of the 2^DB bins, BPT per thread
    constexpr int BPT = (1 << DB) / NT;
    unsigned hv[BPT];
    unsigned hs = 0;
#pragma unroll
    for (int u = 0; u < BPT; ++u) { hv[u] = sm.hist[BPT * threadIdx.x + u]; hs += hv[u]; }
    unsigned x = hs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) sm.wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const unsigned v = sm.wsum[lane];
      unsigned y = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      sm.wsum[lane] = y - v;
    }
    __syncthreads();
    unsigned excl = sm.wsum[wid] + x - hs;
#pragma unroll
    for (int u = 0; u < BPT; ++u) {
      if (excl < need && need <= excl + hv[u]) {
        sm.digit = BPT * threadIdx.x + u; sm.need = need - excl; sm.dcount = hv[u];
      }
      excl += hv[u];
    }
    __syncthreads();
    need = sm.need;
    prefix = (pshift == 32 ? 0u : (prefix << width)) | sm.digit;
    pshift = shift;
    const unsigned dc = sm.dcount;
    __syncthreads();
    if (shift == 0) {
      if (eq_out) *eq_out = dc;
      break;
    }
  }
  *take = need;
  return prefix;
}

// ------------------------------------------------------------------------------------------
// Sampled-bracket selection of the kth smallest key (used by the edge and final selections).
// The radix selection reads all n keys once per 11-bit digit plus once for min/max (4-5 passes
// over data that, per micro-batch, no longer fits L2).  Here: kFsS keys at evenly spaced
// positions are drawn into shared memory, their ranks kth*S/n -/+ kFsMargin give a bracket
// [L, H] (selected among the sample by cta_kth32 on shared memory), one pass counts the keys
// below L and gathers the keys in [L, H] (and their ids) into shared memory, and the kth is
// selected among the gathered keys.  The result is the kth smallest key, the same whatever the
// method: when the bracket misses it or overflows the buffer, the full radix selection runs.
// ------------------------------------------------------------------------------------------
constexpr int kFsS = 4096;                 // sample size
constexpr int kFsMargin = 160;             // bracket half-width in sample ranks (> 5 sigma)
constexpr int kFsCap = 8192;               // gathered keys (and ids) held in shared memory
struct FastSelSmem {
  uint32_t samp[kFsS];
  uint32_t key[kFsCap];
  int id[kFsCap];
  unsigned cnt, below, mn;
};
constexpr size_t kFsSmem = sizeof(FastSelSmem);

// kth smallest of key(i) over i < n (all valid); *take = kth - #(keys < result).  If IDS, the
// gathered ids (idf(i)) of the keys equal to the result are left in fs.key/fs.id[0, fs.cnt) for
// the caller's tie split (fs.cnt = UINT_MAX when the fallback ran).  *min_out = smallest key.
template <bool IDS, typename KeyF, typename IdF>
__device__ uint32_t cta_kth32_bracket(int n, unsigned kth, KeyF key, IdF idf, unsigned* take, FastSelSmem& fs,
                                      Kth32Smem& sm, uint32_t* min_out) {
  constexpr int NT = kSelNT;
  if (n <= 8 * kFsS) {                                // small (<= 32k keys): the radix selection directly
    if (IDS && threadIdx.x == 0) fs.cnt = 0xFFFFFFFFu;
    __syncthreads();
    return cta_kth32(n, kth, [&](int i, bool* ok) { *ok = true; return key(i); }, take, sm, min_out);
  }
  for (int j = threadIdx.x; j < kFsS; j += NT) fs.samp[j] = key((int)(((long long)j * n) / kFsS));
  if (threadIdx.x == 0) { fs.cnt = 0; fs.below = 0; fs.mn = 0xFFFFFFFFu; }
  __syncthreads();
  const long long r = ((long long)kth * kFsS + n - 1) / n;          // expected sample rank (1-based)
  const long long rl = r - kFsMargin, rh = r + kFsMargin;
  unsigned t0;
  const uint32_t L = rl >= 1 ? cta_kth32(kFsS, (unsigned)rl, [&](int i, bool* ok) { *ok = true; return fs.samp[i]; },
                                         &t0, sm) : 0u;
  const uint32_t H = rh <= kFsS ? cta_kth32(kFsS, (unsigned)rh, [&](int i, bool* ok) { *ok = true; return fs.samp[i]; },
                                            &t0, sm) : 0xFFFFFFFFu;
  // one pass: count below L, gather [L, H], minimum
  unsigned below = 0, mn = 0xFFFFFFFFu;
  for (int i = threadIdx.x; i < n; i += NT) {
    const uint32_t k = key(i);
    mn = min(mn, k);
    below += k < L;
    if (k >= L && k <= H) {
      const unsigned at = atomicAdd(&fs.cnt, 1u);
      if (at < kFsCap) {
        fs.key[at] = k;
        if (IDS) fs.id[at] = idf(i);
      }
    }
  }
  below = warp_sum(below);
  mn = warp_min(mn);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&fs.below, below);
    atomicMin(&fs.mn, mn);
  }
  __syncthreads();
  const unsigned cnt = fs.cnt, nb = fs.below;
  if (min_out) *min_out = fs.mn;
  if (cnt > (unsigned)kFsCap || kth <= nb || kth > nb + cnt) {       // bracket missed: full radix
    __syncthreads();
    if (IDS && threadIdx.x == 0) fs.cnt = 0xFFFFFFFFu;
    __syncthreads();
    return cta_kth32(n, kth, [&](int i, bool* ok) { *ok = true; return key(i); }, take, sm, nullptr);
  }
  return cta_kth32((int)cnt, kth - nb, [&](int i, bool* ok) { *ok = true; return fs.key[i]; }, take, sm);
}

// ------------------------------------------------------------------------------------------
// a3  edges: d_min = min of the sample estimates, d_max = budget-th smallest
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelNT) k_select_edges(Batch b, Dev ix) {
  __shared__ Kth32Smem sm;
  extern __shared__ __align__(16) uint8_t fsm[];
  FastSelSmem& fs = *reinterpret_cast<FastSelSmem*>(fsm);
  const int q = blockIdx.x;
  const int ns = b.nsamp[q];
  if (ns == 0) return;
  const int n = b.poff[(size_t)q * (b.nprobe + 1) + ns];
  const float* v = b.val + (size_t)q * b.cap;
  unsigned take;
  uint32_t kmin;
  const uint32_t kmax = cta_kth32_bracket<false>(n, (unsigned)b.budget, [&](int i) { return f2key(v[i]); },
                                                 [&](int i) { return 0; }, &take, fs, sm, &kmin);
  if (threadIdx.x == 0) {
    b.edges[2 * q] = key2f((uint32_t)kmin);
    b.edges[2 * q + 1] = key2f((uint32_t)kmax);
    atomicAdd((unsigned long long*)&b.stats[2], (unsigned long long)n);   // sample objects
  }
}

// ------------------------------------------------------------------------------------------
// f2  Algorithm 4 l.2-4 (reading R22): tau_pred = bucket of the r-th smallest sample
//     estimate, r = max(1, floor(budget * |O_sample| / n_o)).  0 without a sample (nothing early).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelNT) k_tau_pred(Batch b, Dev ix) {
  __shared__ Kth32Smem sm;
  extern __shared__ __align__(16) uint8_t fsm[];
  FastSelSmem& fs = *reinterpret_cast<FastSelSmem*>(fsm);
  const int q = blockIdx.x;
  const int ns = b.nsamp[q];
  if (ns == 0) {
    if (threadIdx.x == 0) b.tpred[q] = 0;
    return;
  }
  const int* po = b.poff + (size_t)q * (b.nprobe + 1);
  const int n = po[ns], ntot = po[b.nprobe];
  const float* v = b.val + (size_t)q * b.cap;
  const long long r = min((long long)n, max(1LL, (b.budget * (long long)n) / max(1, ntot)));
  unsigned take;
  const uint32_t kr = cta_kth32_bracket<false>(n, (unsigned)r, [&](int i) { return f2key(v[i]); },
                                               [&](int i) { return 0; }, &take, fs, sm, nullptr);
  if (threadIdx.x == 0) {
    CellFn cf;
    cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
    b.tpred[q] = cf(key2f(kr));
  }
}

// ------------------------------------------------------------------------------------------
// a5  Update: tau = first cell whose cumulative count reaches the budget (Alg. 1 l.5-11).
//     One warp per query, 8 cells per lane, inclusive scan.  tau = infinity when no sample.
// ------------------------------------------------------------------------------------------
// The n_ew -> m equal-depth remap (Eq. 6 with map; reading R6): the sample's histogram
// over the equal-width cells (its estimates are the first poff[nsamp] entries of val), then the
// greedy equal-depth walk by one thread (256 steps).  One CTA per query.
__global__ void __launch_bounds__(256) k_remap(Batch b) {
  __shared__ int h0[kCells];
  const int q = blockIdx.x;
  const int ns = b.nsamp[q];
  uint8_t* mp = b.rmap + (size_t)q * kCells;
  h0[threadIdx.x] = 0;
  __syncthreads();
  if (ns > 0) {
    CellFn cf;
    cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
    const int n = b.poff[(size_t)q * (b.nprobe + 1) + ns];
    const float* v = b.val + (size_t)q * b.cap;
    for (int i0 = 0; i0 < n; i0 += 256) {
      const int i = i0 + threadIdx.x;
      warp_hist_add(h0, i < n ? cf(v[i]) : 255);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int m = b.remap_m, nb = b.nbuckets;
    long long T = 0;
    for (int c = 0; c < nb; ++c) T += h0[c];
    long long run = 0;
    int bk = 0;
    for (int c = 0; c < kCells; ++c) {
      if (c >= nb) { mp[c] = 255; continue; }
      mp[c] = (uint8_t)bk;
      run += h0[c];
      if (bk < m - 1 && run * m >= (long long)(bk + 1) * T) ++bk;
    }
  }
}

__global__ void __launch_bounds__(32) k_tau(Batch b) {
  const int q = blockIdx.x, lane = threadIdx.x;
  int tau = kTauInf;
  if (b.nsamp[q] > 0 && b.remap_m > 0) {
    // equal-depth buckets: histogram of the buckets, first bucket reaching the budget, then
    // the last cell mapped at or below it ({map[cell] <= tau_b} = {cell <= tau})
    __shared__ long long hb[kCells];
    const int* H = b.hist + (size_t)q * kCells;
    const uint8_t* mp = b.rmap + (size_t)q * kCells;
    for (int i = lane; i < kCells; i += 32) hb[i] = 0;
    __syncwarp();
    if (lane == 0)
      for (int c = 0; c < 255; ++c)
        if (mp[c] < b.remap_m) hb[mp[c]] += H[c];
    __syncwarp();
    if (lane == 0) {
      long long cum = 0;
      int tb = -1;
      for (int i = 0; i < b.remap_m && tb < 0; ++i) {
        cum += hb[i];
        if (cum >= b.budget) tb = i;
      }
      if (tb >= 0) {
        int last = 0;
        for (int c = 0; c < 255; ++c)
          if (mp[c] <= tb) last = c;
        tau = last;
      }
    }
    if (lane == 0) b.tau[q] = tau;
    return;
  }
  if (b.nsamp[q] > 0) {
    const int* H = b.hist + (size_t)q * kCells;
    long long v[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { v[j] = H[lane * 8 + j]; s += v[j]; }
    long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    long long c = incl - s;
    int found = kTauInf;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c += v[j];
      if (c >= b.budget && found == kTauInf) found = lane * 8 + j;
    }
    tau = warp_min(found);    // <= 254 by the sample rule (DESIGN R5)
  }
  if (lane == 0) b.tau[q] = tau;
}

// ------------------------------------------------------------------------------------------
// a6  Collect l.19-21: superset S* = {cell <= tau}, compacted in probe order (deterministic).
//     Chunks of kChunk objects per CTA, 32 per thread (two 16-byte loads of cell ids):
//     k_count -> per-chunk counts, k_chunk_offsets -> per-query exclusive scan, k_emit -> rows.
// ------------------------------------------------------------------------------------------
constexpr int kCmpNT = 256, kPerThr = 32, kChunk = kCmpNT * kPerThr;

struct Cells32 { uint4 a, b; };                      // bucket ids of 32 consecutive elements

// Cell ids of elements [i0, i0 + 32) of query q (ragged tail padded with 255 = never a candidate)
__device__ __forceinline__ Cells32 chunk_load(const Batch& b, int q, int i0, int n) {
  Cells32 x{make_uint4(~0u, ~0u, ~0u, ~0u), make_uint4(~0u, ~0u, ~0u, ~0u)};
  if (i0 >= n) return x;
  const uint8_t* cl = b.cells + (size_t)q * b.cap + i0;
  const int m = min(kPerThr, n - i0);
  if (m == kPerThr) {
    x.a = reinterpret_cast<const uint4*>(cl)[0];
    x.b = reinterpret_cast<const uint4*>(cl)[1];
    return x;
  }
  uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
  for (int e = 0; e < kPerThr; ++e)
    w[e >> 2] |= (e < m ? (uint32_t)cl[e] : 255u) << (8 * (e & 3));
  x.a = make_uint4(w[0], w[1], w[2], w[3]);
  x.b = make_uint4(w[4], w[5], w[6], w[7]);
  return x;
}

// bit e set <=> element i0 + e (e < 32) is a candidate (cell <= tau): eight byte-wise SIMD
// compares, the per-byte results gathered into 4-bit nibbles by one multiply each
__device__ __forceinline__ unsigned chunk_flags(const Cells32& x, int i0, int n, int tau) {
  if (i0 >= n) return 0;
  const int m = min(kPerThr, n - i0);
  const unsigned valid = m == 32 ? 0xffffffffu : ((1u << m) - 1u);
  if (tau == kTauInf) return valid;
  const unsigned t4 = (unsigned)tau * 0x01010101u;   // tau <= 254 here
  const uint32_t w[8] = {x.a.x, x.a.y, x.a.z, x.a.w, x.b.x, x.b.y, x.b.z, x.b.w};
  unsigned f = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const unsigned le = (__vcmpleu4(w[e], t4) >> 7) & 0x01010101u;   // 1 per byte <= tau
    f |= ((le * 0x01020408u) >> 24) << (4 * e);                      // bytes -> bits 0..3
  }
  return f & valid;
}

// Candidate count of kCntPer consecutive chunks per CTA (all loads issued up front).
constexpr int kCntPer = 4;
__global__ void __launch_bounds__(kCmpNT) k_count(Batch b, int* chunk_cnt, int nchunk) {
  __shared__ int red[kCntPer][kCmpNT / 32];
  const int q = blockIdx.y;
  const int n = b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe];
  const int tau = b.tau[q];
  const int need = (n + kChunk - 1) / kChunk;
  // CTA (x, query) takes chunk groups x, x + gridDim.x, ... of the query's real chunks
  for (int c0 = blockIdx.x * kCntPer; c0 < need; c0 += gridDim.x * kCntPer) {
  __syncthreads();                                   // red[] of the previous group read
  Cells32 x[kCntPer];
#pragma unroll
  for (int u = 0; u < kCntPer; ++u)
    x[u] = chunk_load(b, q, (c0 + u) * kChunk + threadIdx.x * kPerThr, tau == kTauInf ? 0 : n);
#pragma unroll
  for (int u = 0; u < kCntPer; ++u) {
    int cnt = __popc(chunk_flags(x[u], (c0 + u) * kChunk + threadIdx.x * kPerThr, n, tau));
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0) red[u][threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x < kCntPer && c0 + (int)threadIdx.x < need) {
    int t = 0;
    for (int w = 0; w < kCmpNT / 32; ++w) t += red[threadIdx.x][w];
    chunk_cnt[(size_t)q * nchunk + c0 + threadIdx.x] = t;
  }
  }
}

__global__ void __launch_bounds__(256) k_chunk_offsets(Batch b, int* chunk_cnt, int nchunk) {
  __shared__ int wsum[8];
  const int q = blockIdx.x;
  int* cc = chunk_cnt + (size_t)q * nchunk;
  const int need = (b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe] + kChunk - 1) / kChunk;
  int run = 0;
  for (int base = 0; base < need; base += 256) {
    const int c = base + threadIdx.x;
    const int v = c < need ? cc[c] : 0;
    int incl = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < 8; ++w) { if (w < wid) pre += wsum[w]; tot += wsum[w]; }
    if (c < need) {
      cc[c] = run + pre + incl - v;
      const int* po = b.poff + (size_t)q * (b.nprobe + 1);
      const int x = c * kChunk;                       // last j with po[j] <= x
      int lo = 0, hi = b.nprobe - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (po[mid] <= x) lo = mid; else hi = mid - 1;
      }
      b.chunkj[(size_t)q * nchunk + c] = lo;
    }
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int n = b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe];
    b.ncand[q] = run;
    atomicAdd((unsigned long long*)&b.stats[0], (unsigned long long)n);
    atomicAdd((unsigned long long*)&b.stats[1], (unsigned long long)run);
  }
}

// One chunk per CTA.  The lists covering the chunk (from chunkj) have their offsets and row
// bases staged in shared memory with one parallel load; a candidate's list is then a
// shared-memory binary search and its row rbase[j] + i.  The chunk's candidate rows are placed
// in shared memory at their block-scan rank, then written out with coalesced stores (the
// original ids are gathered by the re-rank, which reads each candidate's row anyway).  Few dependent global accesses per CTA: the kernel is latency-bound.
constexpr int kEmitWin = 256;                        // lists staged per chunk (else global search); 6 CTAs/SM
struct EmitSmem {
  int wcnt[kCmpNT / 32];
  int s_pre[kCmpNT];
  unsigned s_flg[kCmpNT];
  int s_po[kEmitWin + 1];
  long long s_rb[kEmitWin];
};

// the thread's 32 cell bytes of chunk c (beyond cap: 0xff, masked by chunk_flags anyway)
__device__ __forceinline__ Cells32 emit_cells(const Batch& b, int q, int c) {
  Cells32 cx{make_uint4(~0u, ~0u, ~0u, ~0u), make_uint4(~0u, ~0u, ~0u, ~0u)};
  const int i0 = c * kChunk + threadIdx.x * kPerThr;
  const uint4* cl = reinterpret_cast<const uint4*>(b.cells + (size_t)q * b.cap + i0);
  if (i0 + 16 <= b.cap) cx.a = cl[0];                // cap is a multiple of 16, i0 of 32
  if (i0 + 32 <= b.cap) cx.b = cl[1];
  return cx;
}

// the per-chunk values k_emit loads one chunk ahead: candidate offsets of the chunk and of the
// next one, the probed lists holding their first objects
struct EmitMeta { int cbeg, cnext, jc, jnext; };
__device__ __forceinline__ EmitMeta emit_meta(const Batch& b, const int* chunk_off, int nchunk, int q, int c) {
  const size_t cq = (size_t)q * nchunk + c;
  EmitMeta m;
  m.cbeg = chunk_off[cq];
  m.cnext = c + 1 < nchunk ? chunk_off[cq + 1] : 0;
  m.jc = b.chunkj[cq];
  m.jnext = c + 1 < nchunk ? b.chunkj[cq + 1] : 0;
  return m;
}

// returns the number of candidates of the chunk that took an early distance (EARLY; per thread)
template <bool EARLY>
__device__ __forceinline__ int emit_chunk(const Batch& b, const Dev& ix, const int* chunk_off, int nchunk, int q,
                                           int c, const Cells32& cx, EmitSmem& sm, const EmitMeta& mt) {
  int* wcnt = sm.wcnt;
  int* s_pre = sm.s_pre;
  unsigned* s_flg = sm.s_flg;
  int* s_po = sm.s_po;
  long long* s_rb = sm.s_rb;
  const int nprobe = b.nprobe;
  const int* po = b.poff + (size_t)q * (nprobe + 1);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = c * kChunk + threadIdx.x * kPerThr;
  // Round 1: every load that depends on (q, c) only, issued together (the kernel is bound by
  // dependent-load latency, not bandwidth).  Cell bytes past n are masked by chunk_flags.
  const int n = po[nprobe];
  const int tau = b.tau[q];
  const int ncq = b.ncand[q];
  const int cbeg = mt.cbeg, cnext = mt.cnext, jc = mt.jc, jnext = mt.jnext;
  if (c * kChunk >= n) return 0;
  const int need = (n + kChunk - 1) / kChunk;        // chunks without candidates exit at once
  const int cend = c + 1 < need ? cnext : ncq;
  if (cend == cbeg) return 0;                         // segment starts here: rr_segment
  const long long* rb = b.rbase + (size_t)q * nprobe;
  const int jn = (c + 1) * kChunk < n ? jnext : nprobe - 1;
  const int W = jn - jc + 1;                          // lists touching this chunk
  const bool win = W <= kEmitWin;
  if (win)                                            // round 2: the chunk's list window
    for (int t = threadIdx.x; t < W; t += kCmpNT) {
      s_po[t] = po[jc + t];
      s_rb[t] = rb[jc + t];
      if (t == W - 1) s_po[W] = po[jc + W];
    }
  const unsigned f = chunk_flags(cx, i0, n, tau);
  // exclusive prefix of per-thread counts across the block
  const int mine = __popc(f);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wcnt[wid] = incl;
  __syncthreads();
  int pre = 0;
#pragma unroll
  for (int w = 0; w < kCmpNT / 32; ++w) pre += w < wid ? wcnt[w] : 0;
  int pos = pre + incl - mine;
  int* outp = b.cpos + (size_t)q * b.cap + cbeg;     // candidate rows, written in place
  // Algorithm 4: candidates the main scan pass already gave an exact distance (bucket below
  // tau_pred, position after the sample) take it from b.early and leave with the row complemented
  // (negative): the re-rank then only looks up their ids
  const int tp = EARLY ? b.tpred[q] : 0;
  const int emain = EARLY ? po[b.nsamp[q]] : 0;
  const unsigned fe = EARLY && tp > 0 ? chunk_flags(cx, i0, n, tp - 1) : 0u;   // cell < tau_pred
  int ntaken = 0;
  s_pre[threadIdx.x] = pos;
  s_flg[threadIdx.x] = f;
  if (f) {
    // list of the first candidate: last j with po[j] <= i, then walk forward
    const int ifirst = i0 + __ffs(f) - 1;
    const int* sp = win ? s_po : po + jc;
    const int top = win ? W - 1 : nprobe - 1 - jc;
    int lo = 0, hi = top;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sp[mid] <= ifirst) lo = mid; else hi = mid - 1;
    }
    int j = lo;
    int jend = sp[j + 1];
    long long rbase = win ? s_rb[j] : rb[jc + j];
    for (unsigned r = f; r; r &= r - 1) {
      const int i = i0 + __ffs(r) - 1;
      while (i >= jend) {            // next non-empty list containing i
        ++j;
        jend = sp[j + 1];
        rbase = win ? s_rb[j] : rb[jc + j];
      }
      BBC_CHECK(cbeg + pos < b.cap && rbase + i >= 0 && rbase + i < ix.n_local);
      if (b.a3pos) b.a3pos[(size_t)q * b.cap + cbeg + pos] = i;   // Algorithm 3 (list mode)
      int row = (int)(rbase + i);
      if (EARLY && ((fe >> (i - i0)) & 1u) && i >= emain) {
        b.val[(size_t)q * b.cap + cbeg + pos] = b.early[(size_t)q * b.cap + i];
        row = ~row;
        ++ntaken;
      }
      outp[pos++] = row;
    }
  }
  __syncthreads();
  if (b.sstart) {
    // list-order re-rank: candidates before the start of every pair whose object range starts
    // in this chunk, j in [jlo, jhi) (first j with po[j] >= x0, resp. x1)
    auto P = [&](int j) { return win && j >= jc && j <= jc + W ? s_po[j - jc] : po[j]; };
    const int x0 = c * kChunk, x1 = min(n, x0 + kChunk);
    int jlo = jc, jhi;
    if (P(jlo) < x0) ++jlo;
    else while (jlo > 0 && P(jlo - 1) >= x0) --jlo;  // empty pairs at x0 (rare)
    if (x1 < n) {
      jhi = jn;
      if (P(jhi) < x1) ++jhi;
      else while (jhi > 0 && P(jhi - 1) >= x1) --jhi;
    } else {
      jhi = nprobe;
      while (jhi > 0 && P(jhi - 1) >= n) --jhi;
    }
    int* ss = b.sstart + (size_t)q * nprobe;
    for (int j = jlo + threadIdx.x; j < jhi; j += kCmpNT) {
      const int o = P(j) - x0, th = o / kPerThr, bit = o % kPerThr;
      ss[j] = cbeg + s_pre[th] + __popc(s_flg[th] & ((1u << bit) - 1u));
    }
  }
  return ntaken;
}

// ------------------------------------------------------------------------------------------
// f2  Algorithm 4 l.9-11: the exact distance of every object of the main
// pass whose bucket lies below tau_pred, taken straight after the scan pass has written the
// bucket ids -- before Update and Collect know tau.  CTA (x, query) walks the query's chunks of
// bucket ids past the sample (32 ids per thread, two 16-byte loads; flags by chunk_flags against
// tau_pred - 1); a thread finds the list of its first early object by binary search and walks
// forward; the warp then takes the lanes' early objects four at a time: lane t loads 16 bytes of
// each row (all four loads issued before the arithmetic) and of the query, one warp sum per row,
// stored at the object's probe-order position in b.early for k_emit<EARLY> to hand over.
// (Computing them inside the scan kernel, at the end of each work item, was measured first: the
// few warps that chase row latencies hold the whole CTA at the item's barrier and the extra live
// state spills the lookup loop -- C4 scan 48.7 -> 61.3 ms.)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kCmpNT) k_early_rows(Batch b, Dev ix) {
  const int q = blockIdx.y;
  const int tp = b.tpred[q];
  if (tp <= 0) return;
  const int nprobe = b.nprobe;
  const int* po = b.poff + (size_t)q * (nprobe + 1);
  const int n = po[nprobe];
  const int emain = po[b.nsamp[q]];                  // first object after the sample
  const int need = (n + kChunk - 1) / kChunk;
  const long long* rb = b.rbase + (size_t)q * nprobe;
  const int lane = threadIdx.x & 31;
  const int rowb = ix.raw_u8 ? ix.d : ix.d * 4;
  const int nv = rowb >> 4;
  const uint8_t* raw = static_cast<const uint8_t*>(ix.raw);
  const float* qv = b.Q + (size_t)q * ix.d;
  const bool ipm = ix.metric == BBC_METRIC_IP, u8 = ix.raw_u8 != 0;
  float* out = b.early + (size_t)q * b.cap;
  int cnt = 0;
  const int c0 = emain / kChunk + blockIdx.x;
  Cells32 nx = emit_cells(b, q, c0 < need ? c0 : 0);  // the next chunk's ids load ahead
  for (int c = c0; c < need; c += gridDim.x) {
    const Cells32 cx = nx;
    if (c + (int)gridDim.x < need) nx = emit_cells(b, q, c + gridDim.x);
    const int i0 = c * kChunk + threadIdx.x * kPerThr;
    unsigned f = chunk_flags(cx, i0, n, tp - 1);      // bucket < tau_pred
    if (i0 + kPerThr <= emain) f = 0;                 // the sample's objects are not early (R22)
    else if (i0 < emain) f &= ~((1u << (emain - i0)) - 1u);
    cnt += __popc(f);
    int j = 0, jend = 0;
    long long rbase = 0;
    if (f) {                                          // list of the first early object
      const int ifirst = i0 + __ffs(f) - 1;
      int lo = 0, hi = nprobe - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (po[mid] <= ifirst) lo = mid; else hi = mid - 1;
      }
      j = lo;
      jend = po[j + 1];
      rbase = rb[j];
    }
    while (__any_sync(0xffffffffu, f != 0)) {
      int pos = -1, myrow = 0;
      if (f) {
        pos = i0 + __ffs(f) - 1;
        f &= f - 1;
        while (pos >= jend) {                         // next non-empty list containing pos
          ++j;
          jend = po[j + 1];
          rbase = rb[j];
        }
        myrow = (int)(rbase + pos);
        BBC_CHECK(j < nprobe && myrow >= 0 && myrow < ix.n_local && pos < b.cap);
      }
      unsigned m = __ballot_sync(0xffffffffu, pos >= 0);
      while (m) {                                     // four rows in flight per round
        int src[4], row[4], at[4];
        float a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          src[u] = m ? __ffs(m) - 1 : -1;
          m &= m - 1;                                 // 0 stays 0
          a[u] = 0.f;
          row[u] = __shfl_sync(0xffffffffu, myrow, src[u] & 31);
          at[u] = __shfl_sync(0xffffffffu, pos, src[u] & 31);
        }
        for (int t = lane; t - lane < nv; t += 32) {
          uint4 x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (src[u] >= 0 && t < nv) x[u] = __ldg(reinterpret_cast<const uint4*>(raw + (size_t)row[u] * rowb) + t);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (src[u] >= 0 && t < nv) a[u] = early_part(a[u], x[u], qv, t, u8, ipm);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (src[u] >= 0) {                          // uniform: m is the same in every lane
            const float r = warp_sum(a[u]);
            if (lane == 0) out[at[u]] = ipm ? -r : r;
          }
      }
    }
  }
  cnt = warp_sum(cnt);                                // one counter update per warp
  if (lane == 0 && cnt) atomicAdd((unsigned long long*)&b.stats[5], (unsigned long long)cnt);
}

// CTA (x, query) takes chunks x, x + gridDim.x, ...: the grid covers the queries' real chunks
// without one CTA per chunk of the capacity (most of which, past the query's probed objects, had
// only to exit: C4 ~58 % of 735k CTAs)
template <bool EARLY = false>
__global__ void __launch_bounds__(kCmpNT) k_emit(Batch b, Dev ix, const int* chunk_off, int nchunk) {
  __shared__ EmitSmem sm;
  const int q = blockIdx.y;
  const int n = b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe];
  const int need = (n + kChunk - 1) / kChunk;
  int taken = 0;
  // the next chunk's cells and offsets load ahead
  Cells32 nx = emit_cells(b, q, blockIdx.x);
  EmitMeta nm{0, 0, 0, 0};
  if ((int)blockIdx.x < need) nm = emit_meta(b, chunk_off, nchunk, q, blockIdx.x);
  for (int c = blockIdx.x; c < need; c += gridDim.x) {
    __syncthreads();                                 // shared memory of the previous chunk free
    const Cells32 cx = nx;
    const EmitMeta mt = nm;
    if (c + (int)gridDim.x < need) {
      nx = emit_cells(b, q, c + gridDim.x);
      nm = emit_meta(b, chunk_off, nchunk, q, c + gridDim.x);
    }
    taken += emit_chunk<EARLY>(b, ix, chunk_off, nchunk, q, c, cx, sm, mt);
  }
  if (EARLY) {                                       // one counter update per warp per CTA
    taken = warp_sum(taken);
    if ((threadIdx.x & 31) == 0 && taken) atomicAdd((unsigned long long*)&b.stats[6], (unsigned long long)taken);
  }
}

// ------------------------------------------------------------------------------------------
// a7  exact re-rank.  CTA = (query q, slice of its candidates).  LPC lanes cooperate on one
// candidate row (LPC = 8 for rows <= 1 KB, else 32): each lane holds its share of the query in
// registers and loads its share of the row with 16-byte loads; several warp-steps are unrolled
// so that 8 x 16-byte loads per lane are in flight.  Candidate rows are fetched 32 at a time
// with one coalesced load and broadcast by shuffle.  Writes exact d^2 to val (fp32, FMA order
// of the lane split; tolerance 1e-5 relative to the oracle's fp64).
// ------------------------------------------------------------------------------------------
constexpr int kRrNT = 256;

// The lane's share of query q: fp32 rows keep 4 values per 16-byte chunk (qr), uint8 rows 16
// (qu, MAXV <= 2; else read from L1 per use).
template <bool U8, int LPC, int MAXV>
struct RrQuery {
  static constexpr bool QREG = U8 && MAXV <= 2;
  float qr[MAXV][4];
  float qu[QREG ? MAXV : 1][16];
  const float* qv;
  __device__ __forceinline__ void load(const float* q, int sl, int per, int nv) {
    qv = q;
#pragma unroll
    for (int v = 0; v < MAXV; ++v) {
      const int t = sl + LPC * v;
      if (v < per && t < nv && !U8) {
        const float4 x = reinterpret_cast<const float4*>(qv)[t];
        qr[v][0] = x.x; qr[v][1] = x.y; qr[v][2] = x.z; qr[v][3] = x.w;
      }
    }
    if (QREG) {
#pragma unroll
      for (int v = 0; v < (QREG ? MAXV : 1); ++v) {
        const int t = sl + LPC * v;
        if (v < per && t < nv) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4 x = reinterpret_cast<const float4*>(qv)[4 * t + e];
            qu[v][4 * e] = x.x; qu[v][4 * e + 1] = x.y; qu[v][4 * e + 2] = x.z; qu[v][4 * e + 3] = x.w;
          }
        }
      }
    }
  }
};

// One warp: exact d^2 (IP: -<q, x>) of up to 32 candidates whose rows are cp[0 .. n32); writes
// vv[k] and the original id cid[k].  Rows are fetched with one coalesced load and broadcast by
// shuffle; LPC lanes per row, STEPS rows per lane group in flight.
// ER (Algorithm 4): a complemented (negative) row marks a candidate whose exact d^2 is already in
// vv (computed early by the scan, placed by k_emit): only its id is looked up.
template <bool U8, int LPC, int MAXV, int STEPS, bool IP, bool ER = false>
__device__ __forceinline__ void rr_rows32(const Dev& ix, const RrQuery<U8, LPC, MAXV>& Q,
                                          const int* __restrict__ cp, int n32, float* __restrict__ vv,
                                          int* __restrict__ cid, int lane, int per, int nv, int rowb) {
  constexpr int CPW = 32 / LPC;
  const int sub = lane / LPC, sl = lane % LPC;
  const uint8_t* raw = static_cast<const uint8_t*>(ix.raw);
  const int myrow = lane < n32 ? cp[lane] : 0;
  BBC_CHECK(n32 <= 32 && (ER || myrow >= 0) && (myrow < 0 ? ~myrow : myrow) < ix.n_local);
  for (int k0 = 0; k0 < n32; k0 += CPW * STEPS) {
    uint4 x[STEPS][MAXV];
    int kk[STEPS];
    int idr[STEPS];
    bool done[STEPS];
#pragma unroll
    for (int s = 0; s < STEPS; ++s) {
      kk[s] = k0 + s * CPW + sub;
      const int r0 = __shfl_sync(0xffffffffu, myrow, kk[s] & 31);
      done[s] = ER && r0 < 0;
      const int r = done[s] ? ~r0 : r0;
      idr[s] = (sl == 0 && kk[s] < n32) ? (int)__ldg(ix.ids + r) : 0;   // original id (final select)
      const uint4* rp = reinterpret_cast<const uint4*>(raw + (size_t)r * rowb);
#pragma unroll
      for (int v = 0; v < MAXV; ++v) {
        const int t = sl + LPC * v;
        if (v < per && t < nv && !done[s]) x[s][v] = __ldg(rp + t);
        else if (ER) x[s][v] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int s = 0; s < STEPS; ++s) {
      float acc = 0.f;
#pragma unroll
      for (int v = 0; v < MAXV; ++v) {
        const int t = sl + LPC * v;
        if (v < per && t < nv) {
          if (U8) {
            const uint32_t wv[4] = {x[s][v].x, x[s][v].y, x[s][v].z, x[s][v].w};
#pragma unroll
            for (int h = 0; h < 4; ++h)
#pragma unroll
              for (int by = 0; by < 4; ++by) {
                const float xv = (float)((wv[h] >> (8 * by)) & 255u);
                const float qq = Q.QREG ? Q.qu[Q.QREG ? v : 0][h * 4 + by] : __ldg(Q.qv + t * 16 + h * 4 + by);
                if (IP) acc = fmaf(xv, qq, acc);
                else { const float df = xv - qq; acc = fmaf(df, df, acc); }
              }
          } else if (IP) {
            acc = fmaf(__uint_as_float(x[s][v].x), Q.qr[v][0], acc);
            acc = fmaf(__uint_as_float(x[s][v].y), Q.qr[v][1], acc);
            acc = fmaf(__uint_as_float(x[s][v].z), Q.qr[v][2], acc);
            acc = fmaf(__uint_as_float(x[s][v].w), Q.qr[v][3], acc);
          } else {
            const float a0 = __uint_as_float(x[s][v].x) - Q.qr[v][0], a1 = __uint_as_float(x[s][v].y) - Q.qr[v][1];
            const float a2 = __uint_as_float(x[s][v].z) - Q.qr[v][2], a3 = __uint_as_float(x[s][v].w) - Q.qr[v][3];
            acc = fmaf(a0, a0, acc);
            acc = fmaf(a1, a1, acc);
            acc = fmaf(a2, a2, acc);
            acc = fmaf(a3, a3, acc);
          }
        }
      }
#pragma unroll
      for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (sl == 0 && kk[s] < n32) {
        if (!done[s]) vv[kk[s]] = IP ? -acc : acc;
        cid[kk[s]] = idr[s];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// a7  exact re-rank.  CTA = (query q, slice of its candidates).  LPC lanes cooperate on one
// candidate row (LPC = 8 for rows <= 1 KB, else 32): each lane holds its share of the query in
// registers and loads its share of the row with 16-byte loads; several warp-steps are unrolled
// so that 8 x 16-byte loads per lane are in flight.  Candidate rows are fetched 32 at a time
// with one coalesced load and broadcast by shuffle.  Writes exact d^2 to val (fp32, FMA order
// of the lane split; tolerance 1e-5 relative to the oracle's fp64).
// ------------------------------------------------------------------------------------------
template <bool U8, int LPC, int MAXV, int STEPS, int MINB = 1, bool IP = false, bool ER = false>
__global__ void __launch_bounds__(kRrNT, MINB) k_rerank(Batch b, Dev ix) {
  const int q = b.qperm[blockIdx.y];        // neighbours run together: L2 reuse
  const int lane = threadIdx.x & 31, sl = lane % LPC;
  const int d = ix.d;
  const int rowb = U8 ? d : d * 4;
  const int nv = rowb / 16;
  const int per = (nv + LPC - 1) / LPC;               // <= MAXV (checked by the launcher)
  const int nc = b.ncand[q];
  const int* cp = b.cpos + (size_t)q * b.cap;
  float* vv = b.val + (size_t)q * b.cap;
  int* ci = b.cid + (size_t)q * b.cap;
  RrQuery<U8, LPC, MAXV> Q;
  Q.load(b.Q + (size_t)q * d, sl, per, nv);
  const int gw = blockIdx.x * (kRrNT / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kRrNT / 32);
  for (int cb = gw * 32; cb < nc; cb += nw * 32)      // 32 candidates per warp round
    rr_rows32<U8, LPC, MAXV, STEPS, IP, ER>(ix, Q, cp + cb, min(32, nc - cb), vv + cb, ci + cb, lane, per,
                                            nv, rowb);
}

// ------------------------------------------------------------------------------------------
// a7, list-major order.  The same per-candidate arithmetic as k_rerank, but the work is the
// run of candidates a query has in one inverted list (a "segment"), ordered by list: the warps
// in flight read the rows of a few lists, which every query probing them shares, so the rows
// come from L2 instead of HBM (C3: each row is a candidate of ~20 queries of a batch).
// ------------------------------------------------------------------------------------------
// Candidates of query q before object position P < n: k_emit's count for a chunk with candidates,
// the chunk's offset for an empty one (k_emit exits before writing).
__device__ __forceinline__ int rr_start(const Batch& b, int q, int P, int n, int written) {
  const int nchunk = (int)((b.cap + kChunk - 1) / kChunk);
  const int c = P / kChunk;
  const int need = (n + kChunk - 1) / kChunk;
  const int cb = b.chunk[(size_t)q * nchunk + c];
  const int ce = c + 1 < need ? b.chunk[(size_t)q * nchunk + c + 1] : b.ncand[q];
  return cb == ce ? cb : written;
}

// The segment of pair p = (q, j): candidates [sstart[p], end) where end is the next pair's start
// (ncand after the last pair with objects).  Empty segments are not scheduled.
__device__ __forceinline__ int2 rr_segment(const Batch& b, long long p) {
  const int q = (int)(p / b.nprobe), j = (int)(p % b.nprobe);
  const int* po = b.poff + (size_t)q * (b.nprobe + 1);
  const int n = po[b.nprobe];
  const int P = po[j];
  if (P >= n) return make_int2(0, 0);
  const int s0 = rr_start(b, q, P, n, b.sstart[p]);
  const int s1 = (j + 1 < b.nprobe && po[j + 1] < n) ? rr_start(b, q, po[j + 1], n, b.sstart[p + 1]) : b.ncand[q];
  return make_int2(s0, s1 - s0);
}

// FILL = 0: count the work pieces of every list; FILL = 1: write (q, first, length, 0) of each
// piece at the list's cursor.  One thread per pair; a segment is cut into pieces of at most
// rr_piece candidates so that a warp's work is bounded (segment lengths are heavy-tailed: the
// nearest lists keep most of their objects).
// piece length: 64 candidates, 32 for rows >= 1 KB (C3: 5.68 -> 5.53 ms; C2/C4 unchanged)
__host__ __device__ constexpr int rr_piece(int rowb) { return rowb >= 1024 ? 32 : 64; }
template <bool FILL>
__global__ void __launch_bounds__(256) k_rr_segments(Batch b, int* __restrict__ cnt, int4* __restrict__ seg,
                                                     int piece) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)b.nq * b.nprobe) return;
  const int2 g = rr_segment(b, p);
  if (g.y <= 0) return;
  const int L = b.probe[p];
  const int np = (g.y + piece - 1) / piece;
  if (!FILL) {
    atomicAdd(cnt + L, np);
  } else {
    const int at = atomicAdd(cnt + L, np);
    const int q = (int)(p / b.nprobe);
    for (int i = 0; i < np; ++i)
      seg[at + i] = make_int4(q, g.x + i * piece, min(piece, g.y - i * piece), 0);
  }
}

// Warp w of CTA c takes pieces first + (c * 8 + w) * kRrSPW .. + kRrSPW - 1.  CTAs are
// dispatched in index order and the grid is sized to about the number of pieces, so the pieces
// in flight stay a narrow window of the list order (a persistent grid drifts apart over many
// iterations; a global work counter serialises on one address).  The main launch is single-pass
// (no loop state: no spills at 64 registers); a TAIL launch strides over any pieces beyond its
// coverage (normally none).  nseg = off[nlist], device-side.
template <bool U8, int LPC, int MAXV, int STEPS, int MINB, bool IP, int kRrSPW, bool TAIL, bool ER = false>
__global__ void __launch_bounds__(kRrNT, MINB) k_rerank_seg(Batch b, Dev ix, const int4* __restrict__ seg,
                                                            const int* __restrict__ nseg_p, int first) {
  const int lane = threadIdx.x & 31, sl = lane % LPC;
  const int d = ix.d;
  const int rowb = U8 ? d : d * 4;
  const int nv = rowb / 16;
  const int per = (nv + LPC - 1) / LPC;
  const int nseg = *nseg_p;
  RrQuery<U8, LPC, MAXV> Q;
  int qcur = -1;
  const int stride = gridDim.x * (kRrNT / 32) * kRrSPW;
#pragma unroll 1
  for (int s0 = first + (blockIdx.x * (kRrNT / 32) + (threadIdx.x >> 5)) * kRrSPW; s0 < nseg;
       s0 = TAIL ? s0 + stride : nseg) {
    const int4 mine = lane < kRrSPW && s0 + lane < nseg ? seg[s0 + lane] : make_int4(-1, 0, 0, 0);
#pragma unroll 1
    for (int i = 0; i < kRrSPW; ++i) {
      const int q = __shfl_sync(0xffffffffu, mine.x, i);
      if (q < 0) break;
      const int t0 = __shfl_sync(0xffffffffu, mine.y, i), len = __shfl_sync(0xffffffffu, mine.z, i);
      BBC_CHECK(q < b.nq && t0 >= 0 && len > 0 && t0 + len <= b.ncand[q]);
      if (q != qcur) {
        Q.load(b.Q + (size_t)q * d, sl, per, nv);
        qcur = q;
      }
      const size_t base = (size_t)q * b.cap + t0;
      for (int cb = 0; cb < len; cb += 32)
        rr_rows32<U8, LPC, MAXV, STEPS, IP, ER>(ix, Q, b.cpos + base + cb, min(32, len - cb), b.val + base + cb,
                                                b.cid + base + cb, lane, per, nv, rowb);
    }
  }
}

// ------------------------------------------------------------------------------------------
// a8  final top-k by (exact d^2, id): CTA radix select, then order-preserving write-out.
// ------------------------------------------------------------------------------------------
// a8: final top-k by (exact d^2, id).  The kth smallest d^2 key T is selected first (32-bit
// radix, reading the distances only); the ids are looked at only to split the elements equal
// to T (ties), by a second 32-bit selection among them.  Then an order-preserving write-out.
template <int DB>
__global__ void __launch_bounds__(kSelNT) k_final_select(Batch b, Dev ix, long long* out_ids,
                                                         float* out_d2) {
  // DB = 13 for large candidate sets: the ~25 differing bits of the distances' keys take two
  // histogram passes instead of three (each pass re-reads the query's distances; C4 select
  // 6.01 -> 5.67 ms); small sets keep 11-bit digits (C2: 0.18 vs 0.21 ms, the 8,192-bin
  // histograms' clearing and scan cost more than the pass they save)
  __shared__ Kth32SmemT<DB> sm;
  __shared__ int wcnt[kSelNT / 32 + 1];
  const int q = blockIdx.x;
  const int nc = b.ncand[q];
  BBC_CHECK(nc >= 0 && nc <= b.cap);
  const int k = b.k;
  const int* cp = b.cid + (size_t)q * b.cap;
  const float* vv = b.val + (size_t)q * b.cap;
  long long* oi = out_ids + (size_t)q * k;
  float* od = out_d2 + (size_t)q * k;
  uint32_t T = 0xffffffffu, I = 0xffffffffu;
  bool all = true;
  if (nc > k) {
    // (measured slower here than these radix passes, whose re-reads hit L2 -- the CTAs in
    // flight hold ~100 MB of distances: the sampled bracket, cta_kth32_bracket, C4 select 6.7 ->
    // 7.2 ms; gathering the first digit's bin with its ids into 64 KB of shared memory and
    // finishing there, 6.5 -> 7.2 ms)
    unsigned take, eq;
    T = cta_kth32(nc, (unsigned)k, [&](int i, bool* ok) { *ok = true; return f2key(vv[i]); }, &take, sm,
                  nullptr, &eq);
    // elements equal to T: take the `take` smallest ids (ids are unique) -- unless all of them
    // are taken (no tie across the k-th position, the usual case for real-valued data: the id
    // selection's passes over the candidates are skipped)
    if (take < eq) {
      unsigned t2;
      I = cta_kth32(nc, take, [&](int i, bool* ok) {
            const uint32_t f = f2key(vv[i]);
            *ok = f == T;
            return *ok ? (uint32_t)cp[i] : 0u;
          }, &t2, sm);
    }
    all = false;
  }
  int base = 0;
  for (int t0 = 0; t0 < nc; t0 += kSelNT) {
    const int i = t0 + threadIdx.x;
    bool f = false;
    float dv = 0.f;
    int id = 0;
    if (i < nc) {
      dv = vv[i];
      id = cp[i];
      const uint32_t fk = f2key(dv);
      f = all || fk < T || (fk == T && (uint32_t)id <= I);
    }
    int total;
    int r = block_rank<kSelNT>(f, wcnt, &total);
    if (f && base + r < k) {
      oi[base + r] = (long long)(uint32_t)id;
      od[base + r] = dv;
    }
    base += total;
  }
  for (int i = base + threadIdx.x; i < k; i += kSelNT) {
    oi[i] = -1;
    od[i] = INFINITY;
  }
}

}  // namespace bbc
