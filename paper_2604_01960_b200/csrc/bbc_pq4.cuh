// a2-a4 for 4-bit PQ (the paper's PQ setting, M = d/4 sub-quantizers of 16 centroids, P:L1440;
// SURVEY 8(f) f3), estimated FastScan-style from an 8-bit quantised lookup table:
// DESIGN.md reading R20.  The 16 one-byte LUT entries of a sub-quantizer are four registers,
// and one PRMT (byte permute) looks up four objects at once, so the scan runs on the integer
// ALUs instead of the shared-memory pipe that bounds the 8-bit PQ scan.
//
//   k_pq4_qlut    per query: lo_m, delta, bias and Q[m][c] (uint8) from the fp32 LUT [M x 16].
//   k_pack_codes4 index load: codes regrouped per 32-object group of a list as
//                 [chunk p of 4 sub-quantizers][object octet s = 0..3][4 x 32-bit words], word
//                 mm holding the 4-bit codes of objects 8s..8s+7 for sub-quantizer 4p+mm (nibble
//                 j = object 8s+j).  A group is 16 M bytes; a lane's octet slice of a chunk is 16 B.
//   k_pq4_scan    the scan, work items as k_pq_scan_rq (query, 32768 padded positions): lane l of
//                 warp w handles octet (l & 3) of groups gl + 8i (gl = 32 w + (l >> 2), i < 4,
//                 16 warps, two halves of 512 groups).  Per sub-quantizer and group word w:
//                     s7 = w & 0x77777777, sel = 0x32103210 | ((w >> 1) & 0x44444444)
//                     r1 = prmt(Q[m][0..3], Q[m][4..7], s7)     entries 0-7 (objects 0-3)
//                     r2 = prmt(Q[m][8..11], Q[m][12..15], s7)  entries 8-15
//                     r  = prmt(r1, r2, sel)                    bit 3 of each code
//                 and the same with s7 >> 16, sel >> 16 for objects 4-7; the entries are summed
//                 as 16-bit lanes (even/odd objects), exact (<= 255 M).  est = delta * S + bias.
//                 The scan is bound by the integer ALU pipe (~19 ALU operations per 8 lookups).
#pragma once
#include "bbc_kernels.cuh"

namespace bbc {

constexpr int kQ4NT = 512;                            // 16 warps
constexpr int kQ4Item = 32768;                        // objects per work item
constexpr int kQ4Groups = kQ4Item / 32;               // 1024 groups per work item
constexpr int kQ4GPL = 4;                             // groups per lane per half

// Per query q (one CTA of 32 x M threads... M * 16 <= 1024): Q, delta, bias from the fp32 LUT at
// b.table + q * M * 256 (first M * 16 floats).  Output: uint8 Q at byte offset M * 64 of the same
// per-query area, then (delta, bias) as two floats after it.
__global__ void __launch_bounds__(1024) k_pq4_qlut(Batch b, Dev ix) {
  __shared__ float s_lo[64];
  __shared__ float s_span[32];
  __shared__ float s_db[2];
  const int q = blockIdx.x;
  const int M = ix.M;
  float* lut = b.table + (size_t)q * M * 256;
  uint8_t* qo = reinterpret_cast<uint8_t*>(lut + M * 16);
  const int t = threadIdx.x;                          // entry (m, c) = (t >> 4, t & 15)
  const int lane = t & 31;
  const bool act = t < M * 16;
  const float v = act ? lut[t] : 0.f;
  // row minima and maxima: a row is 16 consecutive lanes
  float mn = v, mx = v;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const float sp = __fsub_rn(mx, mn);                 // max_c LUT - lo_m (exact per row)
  if (act && (lane & 15) == 0) s_lo[t >> 4] = mn;
  float spw = act ? sp : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) spw = fmaxf(spw, __shfl_xor_sync(0xffffffffu, spw, o));
  if (lane == 0) s_span[t >> 5] = spw;
  __syncthreads();
  if (t == 0) {
    float span = 0.f;
    for (int w = 0; w < (M * 16 + 31) / 32; ++w) span = fmaxf(span, s_span[w]);
    float bias = 0.f;
    for (int m = 0; m < M; ++m) bias = __fadd_rn(bias, s_lo[m]);   // m ascending
    s_db[0] = __fdiv_rn(span, 255.0f);
    s_db[1] = bias;
  }
  __syncthreads();
  const float delta = s_db[0];
  if (act) {
    int cq = 0;
    if (delta > 0.f) {
      const float tq = __fdiv_rn(__fsub_rn(v, s_lo[t >> 4]), delta);
      cq = min(255, (int)floorf(__fadd_rn(tq, 0.5f)));
    }
    qo[t] = (uint8_t)cq;
  }
  if (t == 0) {
    float* db = reinterpret_cast<float*>(qo + M * 16);
    db[0] = delta;
    db[1] = s_db[1];
  }
}

// Index load: one CTA per list.
__global__ void __launch_bounds__(256) k_pack_codes4(const uint8_t* __restrict__ codes, const long long* loff,
                                                     const long long* tbase, int M, uint8_t* __restrict__ out) {
  const int L = blockIdx.x;
  const long long r0 = loff[L], n = loff[L + 1] - r0;
  const long long ngroups = (n + 31) / 32;
  const int P = M / 4;
  for (long long u = threadIdx.x; u < ngroups * P * 4; u += blockDim.x) {   // (group, chunk, octet)
    const long long g = u / (P * 4);
    const int p = (int)(u / 4 % P), s = (int)(u % 4);
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const long long x = g * 32 + 8 * s + j;
      if (x >= n) continue;
      const uint8_t* c = codes + (size_t)(r0 + x) * M + 4 * p;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) w[mm] |= (uint32_t)(c[mm] & 15u) << (4 * j);
    }
    *reinterpret_cast<uint4*>(out + tbase[L] + g * 16 * M + p * 64 + s * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ uint32_t imad1(uint32_t x, uint32_t one, uint32_t acc) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(acc));
  return r;
}

// mode 0: sample lists -> estimates (EST); 1: lists [nsamp, nprobe) -> bucket ids; 2: all (debug)
template <int M, bool EST>
__global__ void __launch_bounds__(kQ4NT, 2) k_pq4_scan(Batch b, Dev ix, const uint8_t* __restrict__ codes4,
                                                     const long long* __restrict__ tbase4, float* out_est,
                                                     long long est_stride, int mode, const int2* __restrict__ items,
                                                     const int* __restrict__ nitems) {
  constexpr int P = M / 4;                           // chunks of 4 sub-quantizers
  __shared__ __align__(16) uint8_t s_q[M * 16];
  __shared__ uint32_t gofs[kQ4Groups];                // 16-byte unit of each group
  __shared__ long long gout[kQ4Groups];
  __shared__ int gcnt[kQ4Groups];
  __shared__ int hist[kCells];
  __shared__ int s_popad[kMaxProbe + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nit = *nitems;
  for (int it = blockIdx.x; it < nit; it += gridDim.x) {
    __syncthreads();                                  // shared memory of the previous item free
    const int2 wk = items[it];
    const int q = wk.x;
    const int ns = b.nsamp[q];
    if (mode != 2 && ns == 0) continue;
    const int first = mode == 1 ? ns : 0;
    const int lim = mode == 0 ? ns : b.nprobe;
    const int* popad = b.popad + (size_t)q * (b.nprobe + 1);
    const int nflat = popad[lim];
    const int x0 = popad[first] + wk.y * kQ4Item;
    if (x0 >= nflat) continue;
    for (int j = threadIdx.x; j <= lim; j += kQ4NT) s_popad[j] = popad[j];
    if (!EST)
      for (int i = threadIdx.x; i < kCells; i += kQ4NT) hist[i] = 0;
    const uint8_t* qsrc = reinterpret_cast<const uint8_t*>(b.table + (size_t)q * M * 256 + M * 16);
    for (int i = threadIdx.x; i < M; i += kQ4NT)
      reinterpret_cast<uint4*>(s_q)[i] = reinterpret_cast<const uint4*>(qsrc)[i];
    const float* dbp = reinterpret_cast<const float*>(qsrc + M * 16);
    const float delta = dbp[0], bias = dbp[1];
    const uint32_t one = (uint32_t)(b.nbuckets > 0);   // 1, opaque to the compiler
    __syncthreads();
    const int* po = b.poff + (size_t)q * (b.nprobe + 1);
    const int* pr = b.probe + (size_t)q * b.nprobe;
    const long long obase = EST ? (long long)q * est_stride : (long long)q * b.cap;
    for (int G = threadIdx.x; G < kQ4Groups; G += kQ4NT) {
      uint32_t go = 0;
      long long oo = 0;
      int cnt = 0;
      const int xg = x0 + 32 * G;
      if (xg < nflat) {
        int lo = first, hi = lim - 1;                 // last j with popad[j] <= xg
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_popad[mid] <= xg) lo = mid; else hi = mid - 1;
        }
        const int L = pr[lo];
        const int nL = (int)(ix.loff[L + 1] - ix.loff[L]);
        const int i0 = xg - s_popad[lo];
        cnt = min(32, nL - i0);
        go = (uint32_t)((tbase4[L] + (long long)(i0 >> 5) * 16 * M) >> 4);
        oo = obase + po[lo] + i0;
      }
      gofs[G] = go;
      gout[G] = oo;
      gcnt[G] = cnt;
    }
    __syncthreads();
    CellFn cf;
    if (!EST) cf.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
    const uint4* c16 = reinterpret_cast<const uint4*>(codes4) + (lane & 3);
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      const int gl0 = half * (kQ4Groups / 2) + wid * 32 + (lane >> 2);   // groups gl0 + 8 i
      if (gcnt[half * (kQ4Groups / 2) + wid * 32] == 0) continue;     // warp past the item's objects
      uint32_t acc[kQ4GPL][4];                        // objects (0,2) (1,3) (4,6) (5,7) of the octet
#pragma unroll
      for (int i = 0; i < kQ4GPL; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0u;
      // per chunk: the 4 groups' 16-byte code slices are loaded together, then each
      // sub-quantizer's Q row (one broadcast 16-byte shared load) serves all 4 groups
#pragma unroll 1
      for (int p = 0; p < P; ++p) {
        uint4 cw[kQ4GPL];
#pragma unroll
        for (int i = 0; i < kQ4GPL; ++i) cw[i] = __ldg(c16 + gofs[gl0 + 8 * i] + 4u * (uint32_t)p);
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
          const uint4 lt = reinterpret_cast<const uint4*>(s_q)[4 * p + mm];
#pragma unroll
          for (int i = 0; i < kQ4GPL; ++i) {
            const uint32_t w = mm == 0 ? cw[i].x : mm == 1 ? cw[i].y : mm == 2 ? cw[i].z : cw[i].w;
            const uint32_t s7 = w & 0x77777777u;
            const uint32_t sel = ((w >> 1) & 0x44444444u) | 0x32103210u;
            const uint32_t r = __byte_perm(__byte_perm(lt.x, lt.y, s7), __byte_perm(lt.z, lt.w, s7), sel);
            const uint32_t s7h = s7 >> 16, selh = sel >> 16;
            const uint32_t rh = __byte_perm(__byte_perm(lt.x, lt.y, s7h), __byte_perm(lt.z, lt.w, s7h), selh);
            // the sums as multiply-adds by an opaque 1: they issue on the FMA pipe, not the
            // integer ALU pipe that bounds the scan
            acc[i][0] = imad1(r & 0x00FF00FFu, one, acc[i][0]);
            acc[i][1] = imad1(__byte_perm(r, 0u, 0x4341u), one, acc[i][1]);
            acc[i][2] = imad1(rh & 0x00FF00FFu, one, acc[i][2]);
            acc[i][3] = imad1(__byte_perm(rh, 0u, 0x4341u), one, acc[i][3]);
          }
        }
      }
      // epilogue: lane holds objects 8 (lane & 3) + j of its groups
#pragma unroll
      for (int i = 0; i < kQ4GPL; ++i) {
        const int G = gl0 + 8 * i;
        const int cnt = gcnt[G];
        const long long oo = gout[G] + 8 * (lane & 3);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (8 * (lane & 3) + j < cnt) {
            const uint32_t a2 = acc[i][2 * (j >> 2) + (j & 1)];
            const uint32_t S = (j & 2) ? (a2 >> 16) : (a2 & 0xFFFFu);
            const float est = __fadd_rn(__fmul_rn(delta, (float)S), bias);
            if (EST) {
              out_est[oo + j] = est;
            } else {
              const int cell = cf(est);
              b.cells[oo + j] = (uint8_t)cell;
              if (cell < 255) atomicAdd(&hist[cell], 1);   // plain atomics (see k_pq_scan_rq)
            }
          }
        }
      }
    }
    if (!EST) {
      __syncthreads();
      for (int i = threadIdx.x; i < kCells; i += kQ4NT)
        if (hist[i]) atomicAdd(&b.hist[(size_t)q * kCells + i], hist[i]);
    }
  }
}

}  // namespace bbc
