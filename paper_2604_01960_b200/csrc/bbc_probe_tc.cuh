// a1 coarse probe on the 5th-generation tensor cores (tcgen05, kind::tf32, accumulator in TMEM).
//
// The probe order must be bit-identical to the canonical fp32 d^2, which a
// tensor-core dot product cannot reproduce.  So the tensor cores only *shortlist*:
//
//   1. k_probe_mma: approximate d~(q, c) = |q'|^2 + |c'|^2 - 2 <q', c'> for every (query,
//      centroid), q' = q - mu, c' = c - mu (mu = centroid mean, so the norms stay small), with
//      the dot product in "3xTF32" (x = x_hi + x_lo split, hi*hi + hi*lo + lo*hi on the tensor
//      cores, fp32 accumulation in TMEM).  |d~ - d^2| <= E(q) for every centroid, with
//      E(q) = 2^-12 |q'| c'max + 2^-11 (|q'|^2 + c'max^2)   (derivation there).
//   2. k_probe_select (shortlist mode): T~ = nprobe-th smallest d~; every centroid of the true
//      top-nprobe has d~ <= T~ + 2E (the nprobe smallest d~ all have d^2 <= T~ + E, so the
//      nprobe-th smallest d^2 is <= T~ + E).  The shortlist {d~ <= T~ + 2E} is re-scored with the
//      canonical fp32 d^2 and the nprobe smallest (d^2, list) keys are selected exactly as the
//      SIMT path does: the probe lists are identical by construction.
//
// Kernel shape: CTA = 128 queries x 128 centroids (one UMMA 128x128 accumulator, 128 TMEM
// columns; up to 3 CTAs per SM), K in chunks of 32 (tf32 MMA K = 8, four MMAs x three split products per chunk).
// Operands are staged by the CTA's threads (split into hi/lo while staging) in the canonical
// K-major no-swizzle layout: 8-row x 16-byte core matrices, LBO = 128 B between K-adjacent core
// matrices, SBO = 1 KB between 8-row groups.  One elected thread issues the MMAs; completion is
// tracked with tcgen05.commit on an mbarrier.  Epilogue: tcgen05.ld 32x32b (thread = query row).
#pragma once
#include "bbc_kernels.cuh"

namespace bbc {

constexpr int kTcM = 128, kTcN = 128, kTcKC = 32, kTcNT = 128;
constexpr int kTcSboBytes = (kTcKC / 4) * 128;                // 1 KB per 8-row group
constexpr int kTcABytes = kTcM * kTcKC * 4;                     // 16 KB
constexpr int kTcBBytes = kTcN * kTcKC * 4;                     // 32 KB
constexpr size_t kTcSmem = 2 * kTcABytes + 2 * kTcBBytes + 64;  // hi/lo of A and B + barrier

__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);                      // start address
  d |= (uint64_t)(128u >> 4) << 16;                             // LBO: K-adjacent core matrices
  d |= (uint64_t)((unsigned)kTcSboBytes >> 4) << 32;            // SBO: 8-row groups
  d |= (uint64_t)1 << 46;                                       // descriptor version (sm_100)
  return d;                                                     // base offset 0, SWIZZLE_NONE
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = kTcN
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(kTcIdesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t a, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}

// ---- async-copy and mbarrier helpers (shared with bbc_rbq_tc.cuh)
// K-major, 128-byte swizzle: rows of 128 B, 8-row atoms of 1 KB (SBO), K advanced inside an atom
// by moving the start address (32 B per MMA step)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;                 // SBO: 8-row atoms
  d |= (uint64_t)1 << 46;                            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tma_2d_g2s(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar) : "memory");
}

// bulk global -> shared copy (async proxy) completing on an mbarrier's transaction count
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(a) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t a, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}"
               ::"r"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Stage rows [r0, r0 + R) x K-chunk [k0, k0 + 32) of a row-major fp32 matrix (minus mu) into the
// hi/lo K-major core-matrix layout; rows >= nrows and columns >= d are zero.
template <int R>
__device__ __forceinline__ void tc_stage(const float* __restrict__ X, int nrows, int d, int r0, int k0,
                                         const float* __restrict__ mu, uint8_t* hi, uint8_t* lo) {
  constexpr int kVec = R * (kTcKC / 4);                         // float4 slots
  for (int idx = threadIdx.x; idx < kVec; idx += kTcNT) {
    const int r = idx >> 3, kq = idx & 7;
    const int gr = r0 + r, gk = k0 + 4 * kq;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (gr < nrows) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (gk + e < d) v[e] = X[(size_t)gr * d + gk + e] - mu[gk + e];
    }
    float4 h, l;
    h.x = tf32_hi(v[0]); l.x = v[0] - h.x;
    h.y = tf32_hi(v[1]); l.y = v[1] - h.y;
    h.z = tf32_hi(v[2]); l.z = v[2] - h.z;
    h.w = tf32_hi(v[3]); l.w = v[3] - h.w;
    const int off = (r >> 3) * kTcSboBytes + kq * 128 + (r & 7) * 16;
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

// coarse[q][c] = d~(q, c) for the CTA's 128 x kTcN tile.  cnorm[c] = |c - mu|^2.
__global__ void __launch_bounds__(kTcNT) k_probe_mma(const float* __restrict__ Q, const float* __restrict__ C,
                                                     const float* __restrict__ mu,
                                                     const float* __restrict__ cnorm,
                                                     float* __restrict__ out, int nq, int nlist, int d) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  uint8_t* a_hi = tsm;
  uint8_t* a_lo = a_hi + kTcABytes;
  uint8_t* b_hi = a_lo + kTcABytes;
  uint8_t* b_lo = b_hi + kTcBBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(b_lo + kTcBBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.y * kTcM, c0 = blockIdx.x * kTcN;
  const uint32_t bar_a = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {                                              // kTcN TMEM columns (fp32 128 x kTcN)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
  uint32_t phase = 0;
  const int nk = (d + kTcKC - 1) / kTcKC;
  for (int kc = 0; kc < nk; ++kc) {
    tc_stage<kTcM>(Q, nq, d, q0, kc * kTcKC, mu, a_hi, a_lo);
    tc_stage<kTcN>(C, nlist, d, c0, kc * kTcKC, mu, b_hi, b_lo);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> MMA reads
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int s = 0; s < kTcKC / 8; ++s) {                     // K = 8 per MMA: 2 core matrices
        const uint32_t o = (uint32_t)s * 256u;
        const uint32_t acc0 = (kc | s) ? 1u : 0u;
        tc_mma(tmem, umma_desc_kmajor(al + o), umma_desc_kmajor(bh + o), acc0);
        tc_mma(tmem, umma_desc_kmajor(ah + o), umma_desc_kmajor(bl + o), 1u);
        tc_mma(tmem, umma_desc_kmajor(ah + o), umma_desc_kmajor(bh + o), 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(bar_a) : "memory");
    }
    mbar_wait(bar_a, phase);                                    // MMAs done: smem reusable
    phase ^= 1u;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows = queries), 32 columns at a time
  const int r = warp * 32 + lane;
  const int q = q0 + r;
  float qn = 0.f;
  if (q < nq)
    for (int t = 0; t < d; ++t) {
      const float x = Q[(size_t)q * d + t] - mu[t];
      qn = fmaf(x, x, qn);
    }
  for (int cb = 0; cb < kTcN; cb += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb;
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
    if (q < nq) {
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int c = c0 + cb + e;
        if (c < nlist) out[(size_t)q * nlist + c] = qn + cnorm[c] - 2.0f * __uint_as_float(v[e]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

// ------------------------------------------------------------------ warp-specialised variant
// Same products and the same d~ as k_probe_mma, for d <= 128, as a persistent pipeline:
//   * A = the CTA's 128 centred queries, split hi/lo once into tensor memory (columns 256 + k and
//     384 + k; lane = query), so it is never re-staged across centroid tiles;
//   * B = the centred centroids, split hi/lo once at index load ([nlist_pad x d] each), loaded per
//     (centroid tile, 32-element K chunk) by two TMA copies (128-byte swizzle) into a ring of
//     kPwStages shared-memory stages;
//   * one lane issues the 3 x (d/8) MMAs of a centroid tile (TS: A from TMEM) into one of two
//     128-column accumulators; 4 warps read them out, form d~ = |q'|^2 + |c'|^2 - 2<q', c'> and
//     write the 128 x 128 tile through a padded shared-memory transpose (coalesced rows).
// CTA (query tile qt, stripe s) takes centroid tiles s, s + S, ... (S stripes per query tile).
constexpr int kPwStages = 4, kPwEpi = 4, kPwNT = (kPwEpi + 2) * 32;   // 192 threads
constexpr int kPwStageBytes = 2 * 128 * 128;                            // hi + lo, 128 rows x 128 B
constexpr int kPwTrRow = 129;                                           // padded transpose row (floats)
constexpr size_t kPwSmem = (size_t)kPwStages * kPwStageBytes + (size_t)kPwEpi * 32 * kPwTrRow * 4 + 256;

__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(tmem_d), "r"(tmem_a), "l"(b), "r"(kTcIdesc), "r"(acc));
}

__global__ void __launch_bounds__(kPwNT, 1) k_probe_mma_ws(const float* __restrict__ Q, const float* __restrict__ mu,
                                                          const float* __restrict__ cnorm, float* __restrict__ out,
                                                          int nq, int nlist, int d, int stripes,
                                                          const __grid_constant__ CUtensorMap tmHi,
                                                          const __grid_constant__ CUtensorMap tmLo) {
  extern __shared__ __align__(1024) uint8_t psm[];
  float* tr = reinterpret_cast<float*>(psm + (size_t)kPwStages * kPwStageBytes);   // [4][32][129]
  uint64_t* bars = reinterpret_cast<uint64_t*>(tr + kPwEpi * 32 * kPwTrRow);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kPwStages + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8u * kPwStages;
  const uint32_t accf0 = empty0 + 8u * kPwStages, acce0 = accf0 + 16u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x / stripes, stripe = blockIdx.x % stripes;
  const int q0 = qt * kTcM;
  const int nct = (nlist + kTcN - 1) / kTcN;
  const int ntile = stripe < nct ? (nct - stripe + stripes - 1) / stripes : 0;   // tiles s, s+S, ...
  const int nkc = (d + 31) / 32;
  if (ntile == 0) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPwStages; ++i) {
      mbar_init(full0 + 8u * i, 1);
      mbar_init(empty0 + 8u * i, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(accf0 + 8u * a, 1);
      mbar_init(acce0 + 8u * a, kPwEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tAh = tmem + 256, tAl = tmem + 384;
  float qn = 0.f;
  if (warp < kPwEpi) {
    // A: thread = query row r; q' = q - mu split hi/lo into TMEM (8 columns per store); |q'|^2
    const int r = 32 * warp + lane, q = q0 + r;
    const uint32_t lrow = (uint32_t)(32 * warp) << 16;
    for (int k0 = 0; k0 < 32 * nkc; k0 += 8) {
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int t = k0 + e;
        float x = 0.f;
        if (q < nq && t < d) {
          x = Q[(size_t)q * d + t] - mu[t];
          qn = fmaf(x, x, qn);
        }
        const float h = tf32_hi(x);
        hi[e] = __float_as_uint(h);
        lo[e] = __float_as_uint(x - h);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   ::"r"(tAh + lrow + (uint32_t)k0), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]),
                     "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   ::"r"(tAl + lrow + (uint32_t)k0), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]),
                     "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (warp == kPwEpi) {
    // ---- producer: per (tile, K chunk) two TMA copies (hi, lo: 128 rows x 32 floats each)
    if (lane == 0) {
      int u = 0;
      for (int it = 0; it < ntile; ++it) {
        const int c0 = (stripe + it * stripes) * kTcN;
        for (int kc = 0; kc < nkc; ++kc, ++u) {
          const int st = u % kPwStages;
          if (u >= kPwStages) mbar_wait(empty0 + 8u * st, (unsigned)((u / kPwStages - 1) & 1));
          const uint32_t fb = full0 + 8u * st;
          mbar_arrive_tx(fb, (uint32_t)kPwStageBytes);
          const uint32_t dst = smem_u32(psm + (size_t)st * kPwStageBytes);
          tma_2d_g2s(dst, &tmHi, 32 * kc, c0, fb);
          tma_2d_g2s(dst + kPwStageBytes / 2, &tmLo, 32 * kc, c0, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == kPwEpi + 1) {
    // ---- MMA issuer: per K step (8 elements) lo*hi, hi*lo, hi*hi (the order of k_probe_mma)
    if (lane == 0) {
      int u = 0;
      for (int it = 0; it < ntile; ++it) {
        const int a = it & 1;
        if (it >= 2) mbar_wait(acce0 + 8u * a, (unsigned)((it / 2 - 1) & 1));
        const uint32_t acc = tmem + (uint32_t)(a * kTcN);
        for (int kc = 0; kc < nkc; ++kc, ++u) {
          const int st = u % kPwStages;
          mbar_wait(full0 + 8u * st, (unsigned)((u / kPwStages) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t dh = umma_desc_sw128(smem_u32(psm + (size_t)st * kPwStageBytes));
          const uint64_t dl = umma_desc_sw128(smem_u32(psm + (size_t)st * kPwStageBytes + kPwStageBytes / 2));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int k = 32 * kc + 8 * kk;
            if (k >= d) break;
            const uint32_t o = (uint32_t)kk * 2u;    // 32 B per K step, in 16-byte units
            tc_mma_ts(acc, tAl + (uint32_t)k, dh + o, (kc | kk) ? 1u : 0u);
            tc_mma_ts(acc, tAh + (uint32_t)k, dl + o, 1u);
            tc_mma_ts(acc, tAh + (uint32_t)k, dh + o, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(empty0 + 8u * st) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(accf0 + 8u * a) : "memory");
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: warp w, rows 32w..32w+31; 32 columns at a time through the padded transpose
    float* trw = tr + (size_t)warp * 32 * kPwTrRow;
    for (int it = 0; it < ntile; ++it) {
      const int a = it & 1;
      const int c0 = (stripe + it * stripes) * kTcN;
      mbar_wait(accf0 + 8u * a, (unsigned)((it / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int cb = 0; cb < kTcN; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * kTcN + cb);
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
        if (cb + 32 >= kTcN) {                        // accumulator fully read: free it
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 8u * a);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int c = c0 + cb + e;
          trw[lane * kPwTrRow + e] = qn + (c < nlist ? cnorm[c] : 0.f) - 2.0f * __uint_as_float(v[e]);
        }
        __syncwarp();
        // rows of the warp's 32 queries, 32 consecutive centroids each: one coalesced store per row
        for (int rr = 0; rr < 32; ++rr) {
          const int q = q0 + 32 * warp + rr, c = c0 + cb + lane;
          if (q < nq && c < nlist) out[(size_t)q * nlist + c] = trw[rr * kPwTrRow + lane];
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Index load: centred centroids split hi/lo for the TMA-fed probe ([nlist_pad x d] each, rows
// beyond nlist zero).
__global__ void k_probe_split(const float* __restrict__ C, const float* __restrict__ mu, int nlist, int npad,
                              int d, float* __restrict__ hi, float* __restrict__ lo) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)npad * d) return;
  const int r = (int)(i / d), t = (int)(i % d);
  const float x = r < nlist ? C[(size_t)r * d + t] - mu[t] : 0.f;
  const float h = tf32_hi(x);
  hi[i] = h;
  lo[i] = x - h;
}

}  // namespace bbc
