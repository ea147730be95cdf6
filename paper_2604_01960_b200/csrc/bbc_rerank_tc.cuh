// a7 exact re-rank on the tensor cores (tcgen05, kind::tf32, "3xTF32"), list-major.
//
// The list-order re-rank (k_rerank_seg) reads every candidate's row from L2 once per query that
// has it as a candidate: at C4 a row is a candidate of ~20 queries of a micro-batch and the
// kernel moves 337 GB of rows per step through L2.  Here a CTA takes one inverted list and up to
// 128 of the (query, list) segments that reference it, and computes the dense block
//     D[r][p] = <x_r, q_p>,  rows r of the list (128 per tile)  x  queries p of the segments
// as a tensor-core GEMM (M = 128 rows, N = 128 queries, K = d in chunks of 32).  The block is
// dense while only the candidates are wanted (C4: ~18 % of the (row, query) pairs), but the
// rows are read once per list and chunk of 128 queries instead of once per candidate, and the
// products run on the tensor cores.  The epilogue parks D in shared memory and each segment's
// thread walks its candidates (ascending rows, k_emit's order) tile by tile:
//     L2: val = |x|^2 + |q|^2 - 2 <x, q>      IP: val = -<x, q>
// with |x|^2, |q|^2 as sequential fp32 FMAs.  The dot product is split x = x_hi + x_lo (x_hi =
// the top 19 bits, what the tf32 MMA reads): hi*hi + hi*lo + lo*hi accumulate in fp32 in
// tensor memory (the lo*lo term, < 2^-20 |x||q|, is dropped).  Integer-valued data below 2^11
// has lo = 0 and integer partial sums below 2^24, so its distances are exact, as in the SIMT
// re-rank; otherwise the distance agrees with the fp64 definition within the 1e-5 relative
// tolerance of the re-rank, not bit for bit with the SIMT kernel.
//
// Operands are staged by the CTA's threads in the K-major no-swizzle core-matrix layout of
// bbc_probe_tc.cuh (one K chunk of 32 at a time: A 128 x 32 and B 128 x 32, hi and lo, 64 KB);
// one elected thread issues the MMAs and commits to an mbarrier.  The accumulator block (128
// TMEM columns) is read back in two halves of 64 columns into the (then idle) staging buffer.
#pragma once
#include "bbc_probe_tc.cuh"

namespace bbc {

constexpr int kRtcNT = 128;                        // threads: 4 warps = the 128 TMEM lanes
constexpr int kRtcN = 128;                         // queries (segments) per chunk
constexpr int kRtcDS = 65;                         // padded row stride of the parked D half
constexpr size_t kRtcOffInfo = 2 * kTcABytes + 2 * kTcBBytes;          // 64 KB of operands
constexpr size_t kRtcSmem = kRtcOffInfo + (size_t)kRtcN * 16 + kRtcN * 4 + 128 * 4 + 64;

// Stage K chunk [k0, k0 + 32) of 128 rows given by row(r) (a pointer or nullptr) into hi/lo.
template <bool U8, typename RowF>
__device__ __forceinline__ void rtc_stage(RowF row, int d, int k0, uint8_t* hi, uint8_t* lo) {
  for (int idx = threadIdx.x; idx < 128 * (kTcKC / 4); idx += kRtcNT) {
    const int r = idx >> 3, kq = idx & 7;
    const int gk = k0 + 4 * kq;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const void* p = row(r);
    if (p != nullptr && gk < d) {                   // d % 4 == 0 (checked by the launcher)
      if (U8) {
        const uchar4 u = *reinterpret_cast<const uchar4*>(static_cast<const uint8_t*>(p) + gk);
        v = make_float4((float)u.x, (float)u.y, (float)u.z, (float)u.w);
      } else {
        v = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(p) + gk));
      }
    }
    float4 h, l;
    h.x = tf32_hi(v.x); l.x = v.x - h.x;
    h.y = tf32_hi(v.y); l.y = v.y - h.y;
    h.z = tf32_hi(v.z); l.z = v.z - h.z;
    h.w = tf32_hi(v.w); l.w = v.w - h.w;
    const int off = (r >> 3) * kTcSboBytes + kq * 128 + (r & 7) * 16;
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

// One CTA per inverted list L; seg[off[L] .. off[L+1]) are its segments (q, first, length, 0).
template <bool U8, bool IP>
__global__ void __launch_bounds__(kRtcNT) k_rerank_tc(Batch b, Dev ix, const int4* __restrict__ seg,
                                                      const int* __restrict__ off) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  const int L = blockIdx.x;
  const int s0 = off[L], s1 = off[L + 1];
  if (s0 >= s1) return;
  uint8_t* a_hi = tsm;
  uint8_t* a_lo = a_hi + kTcABytes;
  uint8_t* b_hi = a_lo + kTcABytes;
  uint8_t* b_lo = b_hi + kTcBBytes;
  float* park = reinterpret_cast<float*>(tsm);       // D half [128][kRtcDS], over the operands
  int4* sp = reinterpret_cast<int4*>(tsm + kRtcOffInfo);          // (q, cursor, end, -)
  float* qn = reinterpret_cast<float*>(sp + kRtcN);
  float* xn = qn + kRtcN;
  uint64_t* bar = reinterpret_cast<uint64_t*>(xn + 128);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  int* s_min = reinterpret_cast<int*>(tmem_slot + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_a = smem_u32(bar);
  if (threadIdx.x == 0) {
    mbar_init(bar_a, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(kRtcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
  const int d = ix.d;
  const long long row0 = ix.loff[L];
  const int nL = (int)(ix.loff[L + 1] - row0);
  const size_t rowb = U8 ? (size_t)d : (size_t)d * 4;
  const uint8_t* raw = static_cast<const uint8_t*>(ix.raw) + (size_t)row0 * rowb;
  const int nk = (d + kTcKC - 1) / kTcKC;
  uint32_t phase = 0;
  for (int c0 = s0; c0 < s1; c0 += kRtcN) {
    const int np = min(kRtcN, s1 - c0);
    __syncthreads();                                   // previous chunk's segment table free
    if (threadIdx.x < np) {
      const int4 g = seg[c0 + threadIdx.x];
      sp[threadIdx.x] = make_int4(g.x, g.y, g.y + g.z, 0);
      if (!IP) {
        const float4* qv = reinterpret_cast<const float4*>(b.Q + (size_t)g.x * d);
        float s = 0.f;
        for (int t = 0; t < d / 4; ++t) {
          const float4 x = qv[t];
          s = fmaf(x.x, x.x, s); s = fmaf(x.y, x.y, s); s = fmaf(x.z, x.z, s); s = fmaf(x.w, x.w, s);
        }
        qn[threadIdx.x] = s;
      }
    }
    __syncthreads();
    int t0 = 0;
    while (true) {
      // next tile: the one holding the smallest pending candidate row of the chunk's segments
      if (threadIdx.x == 0) *s_min = nL;
      __syncthreads();
      if (threadIdx.x < np) {
        const int4 g = sp[threadIdx.x];
        if (g.y < g.z) atomicMin(s_min, (int)(b.cpos[(size_t)g.x * b.cap + g.y] - row0));
      }
      __syncthreads();
      const int mn = *s_min;
      if (mn >= nL) break;
      t0 = mn & ~127;
      for (int kc = 0; kc < nk; ++kc) {
        rtc_stage<U8>([&](int r) -> const void* { return t0 + r < nL ? raw + (size_t)(t0 + r) * rowb : nullptr; },
                      d, kc * kTcKC, a_hi, a_lo);
        rtc_stage<false>([&](int r) -> const void* { return r < np ? b.Q + (size_t)sp[r].x * d : nullptr; },
                         d, kc * kTcKC, b_hi, b_lo);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int s = 0; s < kTcKC / 8; ++s) {
            const uint32_t o = (uint32_t)s * 256u;
            const uint32_t acc0 = (kc | s) ? 1u : 0u;
            tc_mma(tmem, umma_desc_kmajor(al + o), umma_desc_kmajor(bh + o), acc0);
            tc_mma(tmem, umma_desc_kmajor(ah + o), umma_desc_kmajor(bl + o), 1u);
            tc_mma(tmem, umma_desc_kmajor(ah + o), umma_desc_kmajor(bh + o), 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(bar_a) : "memory");
        }
        mbar_wait(bar_a, phase);                         // MMAs done: operands reusable
        phase ^= 1u;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // |x|^2 of the tile's rows (thread = row; sequential FMAs)
      if (!IP) {
        const int r = threadIdx.x;
        float s = 0.f;
        if (t0 + r < nL) {
          if (U8) {
            const uint8_t* p = raw + (size_t)(t0 + r) * rowb;
            for (int t = 0; t < d; t += 4) {
              const uchar4 u = *reinterpret_cast<const uchar4*>(p + t);
              s = fmaf((float)u.x, (float)u.x, s); s = fmaf((float)u.y, (float)u.y, s);
              s = fmaf((float)u.z, (float)u.z, s); s = fmaf((float)u.w, (float)u.w, s);
            }
          } else {
            const float4* p = reinterpret_cast<const float4*>(raw + (size_t)(t0 + r) * rowb);
            for (int t = 0; t < d / 4; ++t) {
              const float4 x = __ldg(p + t);
              s = fmaf(x.x, x.x, s); s = fmaf(x.y, x.y, s); s = fmaf(x.z, x.z, s); s = fmaf(x.w, x.w, s);
            }
          }
        }
        xn[r] = s;
      }
      for (int h = 0; h * 64 < np; ++h) {
        // park columns [64h, 64h + 64) of D: warp w holds rows 32w .. 32w + 31
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v[32];
          const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(64 * h + 32 * half);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
              "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
                "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
                "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float* pr = park + (size_t)(warp * 32 + lane) * kRtcDS + 32 * half;
#pragma unroll
          for (int e = 0; e < 32; ++e) pr[e] = __uint_as_float(v[e]);
        }
        __syncthreads();
        // segment threads: the candidates of the tile, in slot order
        const int p = 64 * h + threadIdx.x;
        if (threadIdx.x < 64 && p < np) {
          int4 g = sp[p];
          const size_t base = (size_t)g.x * b.cap;
          const float qq = IP ? 0.f : qn[p];
          while (g.y < g.z) {
            const int r = (int)(b.cpos[base + g.y] - row0) - t0;
            if (r >= 128) break;
            const float dot = park[(size_t)r * kRtcDS + threadIdx.x];
            b.val[base + g.y] = IP ? -dot : fmaf(-2.f, dot, xn[r] + qq);
            b.cid[base + g.y] = (int)__ldg(ix.ids + row0 + t0 + r);
            ++g.y;
          }
          sp[p].y = g.y;
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kRtcN));
}

}  // namespace bbc
