// f1: Algorithm 3, the bound-aware re-rank of IVF+RaBitQ, on the GPU.
//
// Replaces steps a4..a7 of the RaBitQ path when bbc_set_bound_rerank is on.  The codebook is the
// sample's (d_min, d_max) of Algorithm 1 (the same edges the other path uses), and every
// probed object's estimate comes from the RaBitQ scan in EST mode (all probed lists).  Then one
// CTA per query runs, reading R21's one-shot form:
//   A  lb/ub = est -/+ ((2 r_o) r)(t_o eps), t_o = sqrt(1 - g_o^2)(1/g_o), eps = eps0/sqrt(D - 1)
//      (the RaBitQ bound, eps0 P:L1440), fp32 with explicit roundings in that order;
//      their bucket ids a_lb, a_ub (Eq. 6, the canonical CellFn); histograms of both.
//   B  tau = Update(B_u, k): the first bucket whose cumulative a_ub count reaches k;
//      candidates {a_lb <= tau} (B_l plus B_u, l.7-11) gathered grouped by a_lb, and the B_u
//      members (a_ub <= tau) indexed grouped by a_ub.
//   C  l.12-21: i = first non-empty B_l bucket, j = tau; while i < j: exact d^2 of B_l[i] and
//      B_u[j] (an object once), He[cell(exact)]++, j = first bucket where B_u + He reach k,
//      i = next non-empty B_l bucket; then the leftovers of B_u[j] (l.22).
// Re-ranked candidates keep their exact d^2 in val, the others +inf, so k_final_select returns
// the k smallest (exact d^2, id) of B_exact (l.22-23).  With tau = infinity (fewer than k upper
// bounds below d_max) every object with a_lb <= 254 is re-ranked.
#pragma once
#include "bbc_kernels.cuh"

namespace bbc {

#ifndef BBC_A3_NR
#define BBC_A3_NR 2      // rows per warp in flight in the marginal-bucket gathers
#endif
#ifndef BBC_A3_V
#define BBC_A3_V 2       // 16-byte vectors per lane per row per load round
#endif
#ifndef BBC_A3_MINB
#define BBC_A3_MINB 2    // CTAs per SM (register cap)
#endif
constexpr int kA3NT = 512;

struct Alg3Smem {
  int hl[kCells];        // objects not yet re-ranked, by a_lb
  int hu[kCells];        // objects not yet re-ranked, by a_ub
  int he[kCells];        // re-ranked objects, by the bucket of their exact d^2
  int lst[kCells + 1];   // candidate slots grouped by a_lb: bucket c = [lst[c], lst[c+1])
  int ust[kCells + 1];   // B_u index grouped by a_ub
  int lcur[kCells], ucur[kCells];
  int i, j, tau;
};

// every probed list (warp-strided): for each probe-order position p of the list, v = ld(p, row)
// for U positions per lane first (their loads in flight together), then use(p, row, rq2, v)
template <int U, typename LdF, typename UseF>
__device__ __forceinline__ void a3_for_probed(const Batch& b, int q, LdF ld, UseF use) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int* po = b.poff + (size_t)q * (b.nprobe + 1);
  for (int j = w; j < b.nprobe; j += kA3NT / 32) {
    const int p0 = po[j], p1 = po[j + 1];
    const long long rb = b.rbase[(size_t)q * b.nprobe + j];
    const float rq2 = b.rq2[(size_t)q * b.nprobe + j];
    for (int pb = p0 + lane; pb < p1; pb += 32 * U) {
      decltype(ld(0, 0LL)) v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pb + 32 * u < p1) v[u] = ld(pb + 32 * u, rb + pb + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (pb + 32 * u < p1) use(pb + 32 * u, rb + pb + 32 * u, rq2, v[u]);
    }
  }
}

// exact ||q - x||^2 of NR rows by one warp (rows[r] < 0: skipped, returns 0), all lanes return
// them; every row's loads are issued before any arithmetic (16-byte loads for fp32 rows, 4-byte
// for u8, when d is a multiple of 4), so up to NR x 4 loads per lane are in flight -- the
// gathers are latency-bound (ncu: long-scoreboard stalls on the row loads)
template <bool U8, int NR>
__device__ __forceinline__ void a3_exact(const Dev& ix, const float* sq, const long long* rows, int lane,
                                         float* out) {
  const int d = ix.d;
  float acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.f;
  if ((d & 3) == 0) {
    const int nv = d >> 2;
    for (int t0 = 0; t0 < nv; t0 += 32 * BBC_A3_V) {     // BBC_A3_V vectors per lane per row per round
      float4 x[NR][BBC_A3_V];
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int v = 0; v < BBC_A3_V; ++v) {
          const int t = t0 + lane + 32 * v;
          if (rows[r] >= 0 && t < nv) {
            if (U8) {
              const uint32_t w4 = __ldg(reinterpret_cast<const uint32_t*>(
                                            static_cast<const uint8_t*>(ix.raw) + (size_t)rows[r] * d) + t);
              x[r][v] = make_float4((float)(w4 & 255u), (float)((w4 >> 8) & 255u),
                                    (float)((w4 >> 16) & 255u), (float)(w4 >> 24));
            } else {
              x[r][v] = __ldg(reinterpret_cast<const float4*>(
                                  static_cast<const float*>(ix.raw) + (size_t)rows[r] * d) + t);
            }
          }
        }
#pragma unroll
      for (int v = 0; v < BBC_A3_V; ++v) {
        const int t = t0 + lane + 32 * v;
        if (t < nv) {
          const float4 qv = reinterpret_cast<const float4*>(sq)[t];
#pragma unroll
          for (int r = 0; r < NR; ++r)
            if (rows[r] >= 0) {
              const float d0 = x[r][v].x - qv.x, d1 = x[r][v].y - qv.y;
              const float d2 = x[r][v].z - qv.z, d3 = x[r][v].w - qv.w;
              acc[r] = fmaf(d0, d0, acc[r]); acc[r] = fmaf(d1, d1, acc[r]);
              acc[r] = fmaf(d2, d2, acc[r]); acc[r] = fmaf(d3, d3, acc[r]);
            }
        }
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (rows[r] >= 0)
        for (int t = lane; t < d; t += 32) {
          const float xv = U8 ? (float)__ldg(static_cast<const uint8_t*>(ix.raw) + (size_t)rows[r] * d + t)
                              : __ldg(static_cast<const float*>(ix.raw) + (size_t)rows[r] * d + t);
          const float df = xv - sq[t];
          acc[r] = fmaf(df, df, acc[r]);
        }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) out[r] = warp_sum(acc[r]);
}

// warp 0: first c in [0, 255) whose cumulative count (hu[c] for c <= tau, + he[c]) reaches k
__device__ __forceinline__ int a3_threshold(const Alg3Smem& sm, int tau, long long k) {
  const int lane = threadIdx.x & 31;
  long long v[8], s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = lane * 8 + e;
    v[e] = c < 255 ? (long long)(c <= tau ? sm.hu[c] : 0) + sm.he[c] : 0;
    s += v[e];
  }
  long long incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  long long c = incl - s;
  int found = kTauInf;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    c += v[e];
    if (c >= k && found == kTauInf) found = lane * 8 + e;
  }
  return warp_min(found);
}

// warp 0: first non-empty B_l bucket in [0, tau], kTauInf if none
__device__ __forceinline__ int a3_first_nonempty(const Alg3Smem& sm, int tau) {
  const int lane = threadIdx.x & 31;
  int found = kTauInf;
  for (int c = lane; c <= tau; c += 32)
    if (sm.hl[c] > 0) { found = c; break; }
  return warp_min(found);
}

// MODE 0 (BBC_ALG3_QUERY): the whole algorithm, rows gathered by the query's CTA as the loop
// reaches them.  MODE 1 (BBC_ALG3_LIST, first kernel): phase A only; writes each position's a_lb
// to cells, tau to a3tau and the compaction bound (tau, or 254 for tau = infinity) to tau, so
// that k_count/k_emit gather the candidates {a_lb <= tau} in probe order for the list-order
// re-rank; k_alg3_loop then runs the loop on those exact distances.
template <bool U8, int MODE>
__global__ void __launch_bounds__(kA3NT, BBC_A3_MINB) k_alg3(Batch b, Dev ix, float eps0) {
  extern __shared__ __align__(16) float sq[];          // the query, [d]
  __shared__ Alg3Smem sm;
  // queries in locality order (k_qperm): CTAs in flight share probed lists, so candidate rows
  // recur in L2
  const int q = b.qperm[blockIdx.x], tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = kA3NT / 32;
  if (MODE == 0)
    for (int t = tid; t < ix.d; t += kA3NT) sq[t] = b.Q[(size_t)q * ix.d + t];
  for (int c = tid; c < kCells; c += kA3NT) { sm.hl[c] = 0; sm.hu[c] = 0; sm.he[c] = 0; }
  CellFn cf;
  if (b.nsamp[q] > 0) cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
  else cf.init(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), b.nbuckets);   // no sample: all 0
  const float eps = __fdiv_rn(eps0, __fsqrt_rn((float)(ix.D - 1)));
  float* val = b.val + (size_t)q * b.cap;
  uint16_t* lp = b.a3lb + (size_t)q * b.cap;
  __syncthreads();

  // A: bounds and their bucket ids (est is read from val before anything overwrites it)
  a3_for_probed<2>(b, q, [&](int p, long long row) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(ix.factors) + row);
    return make_float3(val[p], f.x, f.y);
  }, [&](int p, long long row, float rq2, float3 v) {
    const float est = v.x, ro = v.y, g = v.z;
    const float r = __fsqrt_rn(rq2);
    const float t = __fmul_rn(__fsqrt_rn(__fsub_rn(1.f, __fmul_rn(g, g))), __fdiv_rn(1.f, g));
    const float delta = __fmul_rn(__fmul_rn(__fmul_rn(2.f, ro), r), __fmul_rn(t, eps));
    const int al = cf(__fsub_rn(est, delta)), au = cf(__fadd_rn(est, delta));
    lp[p] = (uint16_t)(al | (au << 8));
    if (MODE == 1) b.cells[(size_t)q * b.cap + p] = (uint8_t)al;
    if (al < 255) atomicAdd(&sm.hl[al], 1);
    if (au < 255) atomicAdd(&sm.hu[au], 1);
  });
  __syncthreads();
  if (w == 0) {
    const int tau = a3_threshold(sm, 254, b.k);
    if (lane == 0) sm.tau = tau;
  }
  __syncthreads();
  const int tau = sm.tau;
  const int tc = tau == kTauInf ? 254 : tau;             // candidates: a_lb <= tc
  for (int c = tid; c < kCells; c += kA3NT) b.hist[(size_t)q * kCells + c] = c < 255 ? sm.hu[c] : 0;
  if (MODE == 1) {
    if (tid == 0) {
      b.a3tau[q] = tau;
      b.tau[q] = tc;
    }
    return;
  }
  if (tid == 0) {
    int s = 0, u = 0;
    for (int c = 0; c <= tc; ++c) {
      sm.lst[c] = s; sm.lcur[c] = s; s += sm.hl[c];
      sm.ust[c] = u; sm.ucur[c] = u; u += (tau != kTauInf) ? sm.hu[c] : 0;
    }
    sm.lst[tc + 1] = s;
    sm.ust[tc + 1] = u;
  }
  __syncthreads();
  const int nc = sm.lst[tc + 1];

  // B: gather the candidates grouped by a_lb; index B_u grouped by a_ub
  int* cpos = b.cpos + (size_t)q * b.cap;
  int* cid = b.cid + (size_t)q * b.cap;
  uint16_t* lc = b.a3lc + (size_t)q * b.cap;
  int* ordu = b.a3ordu + (size_t)q * b.cap;
  a3_for_probed<2>(b, q, [&](int p, long long) { return (int)lp[p]; },
                   [&](int p, long long row, float, int v) {
    const int al = v & 255, au = v >> 8;
    if (al <= tc) {
      const int c = atomicAdd(&sm.lcur[al], 1);
      BBC_CHECK(c < nc && nc <= b.cap);
      cpos[c] = (int)row;
      cid[c] = (int)__ldg(ix.ids + row);
      lc[c] = (uint16_t)v;
      if (tau != kTauInf && au <= tau) ordu[atomicAdd(&sm.ucur[au], 1)] = c;
    }
  });
  __syncthreads();
  const float kNaN = __int_as_float(0x7fc00000);
  for (int c = tid; c < nc; c += kA3NT) val[c] = kNaN;   // NaN: not re-ranked yet
  __syncthreads();

  // warps re-rank the not-yet-done candidates of a slot range (B_l[i]: slots; B_u[j]: ordu
  // entries), two rows per warp in flight; counts move from B_l / B_u to He
  auto rerank_range = [&](int x0, int x1, const int* map, bool count) {
    constexpr int NR = BBC_A3_NR;
    for (int x = x0 + NR * w; x < x1; x += NR * NW) {
      int c[NR];
      long long rw[NR];
      bool any = false;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        c[r] = x + r < x1 ? (map ? map[x + r] : x + r) : -1;
        BBC_CHECK(c[r] < nc && (c[r] < 0 || (cpos[c[r]] >= 0 && cpos[c[r]] < ix.n_local)));
        rw[r] = (c[r] >= 0 && isnan(val[c[r]])) ? (long long)cpos[c[r]] : -1;   // warp-uniform
        any |= rw[r] >= 0;
      }
      if (!any) continue;
      float d2[NR];
      a3_exact<U8, NR>(ix, sq, rw, lane, d2);
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (rw[r] < 0) continue;
          val[c[r]] = d2[r];
          if (count) {
            const int v = lc[c[r]], al = v & 255, au = v >> 8;
            atomicSub(&sm.hl[al], 1);
            if (au <= tau) atomicSub(&sm.hu[au], 1);
            const int ce = cf(d2[r]);
            if (ce < 255) atomicAdd(&sm.he[ce], 1);
          }
        }
    }
  };
  if (tau == kTauInf) {
    rerank_range(0, nc, nullptr, false);
  } else {
    if (w == 0) {
      const int i0 = a3_first_nonempty(sm, tau);
      if (lane == 0) { sm.i = i0; sm.j = tau; }
    }
    __syncthreads();
    int i = sm.i, j = sm.j;
    while (i < j) {
      rerank_range(sm.lst[i], sm.lst[i + 1], nullptr, true);
      __syncthreads();
      if (j <= tau) rerank_range(sm.ust[j], sm.ust[j + 1], ordu, true);
      __syncthreads();
      if (w == 0) {
        const int j2 = a3_threshold(sm, tau, b.k);
        const int i2 = a3_first_nonempty(sm, tau);
        if (lane == 0) { sm.i = i2; sm.j = j2; }
      }
      __syncthreads();
      i = sm.i;
      j = sm.j;
    }
    if (j <= tau) rerank_range(sm.ust[j], sm.ust[j + 1], ordu, false);   // l.22: threshold bucket's leftovers
  }
  __syncthreads();
  int mine = 0;
  for (int c = tid; c < nc; c += kA3NT) {
    if (isnan(val[c])) val[c] = __int_as_float(0x7f800000);   // not in B_exact: +inf
    else ++mine;
  }
  mine = warp_sum(mine);
  if (lane == 0) atomicAdd(&sm.he[255], mine);           // rows re-ranked (he[255] is unused above)
  __syncthreads();
  if (tid == 0) {
    b.ncand[q] = nc;
    b.tau[q] = tau;
    const int n_o = b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe];
    atomicAdd((unsigned long long*)&b.stats[0], (unsigned long long)n_o);
    atomicAdd((unsigned long long*)&b.stats[1], (unsigned long long)sm.he[255]);
  }
}

// BBC_ALG3_LIST, second kernel: the loop of l.12-21 over the candidates' exact distances, which
// the list-order re-rank has computed for every candidate {a_lb <= tau} (val, probe order).  One
// CTA per query: each candidate's bucket pair from its probe position (a3pos, written by k_emit),
// the counts B_l / B_u, the candidates grouped by a_lb and B_u's by a_ub, then the loop moving
// the counts of B_l[i] and B_u[j] to He (a thread per object, no row gathers); the candidates the
// loop never reaches leave B_exact (+inf), exactly as in MODE 0.
__global__ void __launch_bounds__(kA3NT) k_alg3_loop(Batch b, Dev ix) {
  __shared__ Alg3Smem sm;
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int tau = b.a3tau[q];
  const int tc = tau == kTauInf ? 254 : tau;
  const int nc = b.ncand[q];
  if (tid == 0) b.tau[q] = tau;                          // the threshold, as MODE 0 reports it
  if (tau == kTauInf) return;                            // every candidate is re-ranked
  for (int c = tid; c < kCells; c += kA3NT) { sm.hl[c] = 0; sm.hu[c] = 0; sm.he[c] = 0; }
  CellFn cf;
  if (b.nsamp[q] > 0) cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
  else cf.init(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), b.nbuckets);
  float* val = b.val + (size_t)q * b.cap;
  int* pos = b.a3pos + (size_t)q * b.cap;                // read, then reused as the B_l index
  uint16_t* lc = b.a3lc + (size_t)q * b.cap;
  int* ordu = b.a3ordu + (size_t)q * b.cap;
  uint8_t* done = b.cells + (size_t)q * b.cap;           // per candidate (the cells are consumed)
  const uint16_t* lp = b.a3lb + (size_t)q * b.cap;
  __syncthreads();
  for (int c = tid; c < nc; c += kA3NT) {
    BBC_CHECK(pos[c] >= 0 && pos[c] < b.cap);
    const int v = lp[pos[c]], al = v & 255, au = v >> 8;
    BBC_CHECK(al <= tc);
    lc[c] = (uint16_t)v;
    atomicAdd(&sm.hl[al], 1);
    if (au <= tau) atomicAdd(&sm.hu[au], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int s = 0, u = 0;
    for (int c = 0; c <= tc; ++c) {
      sm.lst[c] = s; sm.lcur[c] = s; s += sm.hl[c];
      sm.ust[c] = u; sm.ucur[c] = u; u += sm.hu[c];
    }
    sm.lst[tc + 1] = s;
    sm.ust[tc + 1] = u;
  }
  __syncthreads();
  for (int c = tid; c < nc; c += kA3NT) {
    const int v = lc[c], al = v & 255, au = v >> 8;
    pos[atomicAdd(&sm.lcur[al], 1)] = c;
    if (au <= tau) ordu[atomicAdd(&sm.ucur[au], 1)] = c;
    done[c] = 0;
  }
  __syncthreads();
  auto visit = [&](int x0, int x1, const int* map, bool count) {
    for (int x = x0 + tid; x < x1; x += kA3NT) {
      const int c = map[x];
      if (done[c]) continue;
      done[c] = 1;
      if (count) {
        const int v = lc[c], al = v & 255, au = v >> 8;
        atomicSub(&sm.hl[al], 1);
        if (au <= tau) atomicSub(&sm.hu[au], 1);
        const int ce = cf(val[c]);
        if (ce < 255) atomicAdd(&sm.he[ce], 1);
      }
    }
  };
  if (w == 0) {
    const int i0 = a3_first_nonempty(sm, tau);
    if (lane == 0) { sm.i = i0; sm.j = tau; }
  }
  __syncthreads();
  int i = sm.i, j = sm.j;
  while (i < j) {
    visit(sm.lst[i], sm.lst[i + 1], pos, true);
    __syncthreads();
    if (j <= tau) visit(sm.ust[j], sm.ust[j + 1], ordu, true);
    __syncthreads();
    if (w == 0) {
      const int j2 = a3_threshold(sm, tau, b.k);
      const int i2 = a3_first_nonempty(sm, tau);
      if (lane == 0) { sm.i = i2; sm.j = j2; }
    }
    __syncthreads();
    i = sm.i;
    j = sm.j;
  }
  if (j <= tau) visit(sm.ust[j], sm.ust[j + 1], ordu, false);   // l.22
  __syncthreads();
  for (int c = tid; c < nc; c += kA3NT)
    if (!done[c]) val[c] = __int_as_float(0x7f800000);          // not in B_exact: +inf
}

__global__ void k_fill_int(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace bbc
