// a3/a4 RaBitQ estimated distances on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// The RaBitQ estimator of object x in list L for query q needs ip = <bits_x, qbar_{q,L}>, the
// inner product of x's 1-bit code with the 4-bit query code of the pair (q, L) (B_q = 4,
// P:L1440).  The SIMT kernel (k_rbq_scan) forms it with 4 popcounts per 32 code
// bits per pair, which is popcount-bound.  Here the work is regrouped list-major: for list L,
// every query that probes it is gathered (inverted probe index), and
//      IP[objects x queries] = bits[objects x D] . qbar[queries x D]^T
// is one integer GEMM on the tensor cores (A = code bits expanded to bytes 0/1, B = 4-bit query
// codes as bytes 0..15, exact int32 accumulation in TMEM).  ip is exact, so every estimate is
// bit-identical to the SIMT kernel's (same fp32 expression tree afterwards).
//
//   k_rbq_l*      : the pair layout: pairs grouped by list (sample pairs j < nsamp first),
//                   each list's slot range padded to a multiple of kRbN (one MMA query tile).
//   k_rbq_pairs   : per (query, probed list): q' = (u - w_L)/r, v_l, Delta, qbar (bytes), s_q,
//                   and (c1, c2, c3, r) -- the canonical per-pair part of the estimator, at the
//                   pair's slot (codes row-major, coalesced).
//   k_rbq_mma_ws  : CTA = (list L, tile of 128 objects); A (the objects' bits as bytes 0/1)
//                   written once into tensor memory, then for each tile of kRbN = 96 pairs: B
//                   (96 x D bytes, TMA tensor copies with 128-byte swizzle, one per 128-byte K
//                   block) + records (bulk copy) into a ring of stages (mbarrier complete_tx),
//                   D/32 MMAs (M=128, N=96, K=32, A from TMEM) into one of two TMEM accumulators,
//                   epilogue by 24 warps: estimate (sample pass) or bucket id (Push).
//   k_cell_hist   : Push histogram per query from its bucket ids (query-major, shared-memory
//                   counts, one global flush per CTA: list-major partial histograms would need
//                   a global atomic per (pair, bucket)).
// Operands, K-major: A (object bits as bytes 0/1) in tensor memory, lane = object, 4 K bytes per
// 32-bit column; B (query codes, TMA) in shared memory as 128-byte-swizzled K blocks of kRbN rows
// x 128 B, SBO = 1 KB (8-row atoms).
#pragma once
#include "bbc_probe_tc.cuh"

namespace bbc {

constexpr int kRbM = 128, kRbN = 96;   // object tile x query tile of one MMA

struct __align__(16) RbqPair {   // per (query, probed list), written by k_rbq_pairs
  float c1, c2, c3, r;
  float rq2;
  int q;
  long long obase;       // q * cap + poff[q][j]: probe-order position of the list's object 0
  // the query's bucket function (Eq. 6, R3), filled by k_rbq_paircell once the edges are known
  float dmin, dmax, inv, bmax;
  int degen, pad0, pad1, pad2;
};
static_assert(sizeof(RbqPair) == 64, "four 16-byte copies per pair");


// Packed fp32 pairs (sm_100 FADD2/FMUL2): each half is the IEEE round-to-nearest (or, for
// add_rm2, round-down) result of its own operands -- element by element the same arithmetic as
// the scalar intrinsics, half the instructions.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long a) {
  float2 r;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(a));
  return r;
}
__device__ __forceinline__ unsigned long long sub_rn2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul_rn2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long add_rn2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long add_rm2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// ------------------------------------------------------------------ per-pair query codes
// CTA = (query, kPairsPerCta consecutive probes): the query's rotated vector u is staged once in
// shared memory; each warp computes kPairsPerWarp pairs (lane holds dims 4 (lane + 32 m) .. +3 of
// q'), their metadata loaded up front by lanes 0..kPairsPerWarp-1.
constexpr int kPairsPerWarp = 8, kPairsPerCta = 8 * kPairsPerWarp;
__global__ void __launch_bounds__(256, 4) k_rbq_pairs(Batch b, Dev ix, const int* __restrict__ islot,
                                                   uint8_t* __restrict__ qbar, RbqPair* __restrict__ pinfo) {
  extern __shared__ __align__(16) float su[];          // [D]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int q = blockIdx.y;
  const int D = ix.D;
  const int D4 = D / 4;                               // float4 slots; lane holds slots lane + 32 m
  constexpr int kMaxM4 = 8;                           // D <= 1024
  for (int i = threadIdx.x; i < D4; i += 256)
    reinterpret_cast<float4*>(su)[i] = reinterpret_cast<const float4*>(b.table + (size_t)q * D)[i];
  __syncthreads();
  const float4* u4 = reinterpret_cast<const float4*>(su);
  const float sD = __fsqrt_rn((float)D);
  // the warp's pairs' metadata, loaded up front by lanes 0..kPairsPerWarp-1
  const int j0 = blockIdx.x * kPairsPerCta + wid * kPairsPerWarp;
  int m_slot = -1, m_L = 0, m_poff = 0;
  float m_rq2 = 0.f;
  if (lane < kPairsPerWarp && j0 + lane < b.nprobe) {
    const long long p = (long long)q * b.nprobe + j0 + lane;
    m_slot = islot[p];
    m_L = b.probe[p];
    m_rq2 = b.rq2[p];
    m_poff = b.poff[(size_t)q * (b.nprobe + 1) + j0 + lane];
  }
  for (int jj = 0; jj < kPairsPerWarp; ++jj) {
    const int slot = __shfl_sync(0xffffffffu, m_slot, jj);
    if (slot < 0) continue;                           // not estimated on this shard / pass (or j >= nprobe)
    const int L = __shfl_sync(0xffffffffu, m_L, jj);
    const float rq2 = __shfl_sync(0xffffffffu, m_rq2, jj);
    const int poff = __shfl_sync(0xffffffffu, m_poff, jj);
    const float r = __fsqrt_rn(rq2);
    const float rinv = r > 0.f ? __fdiv_rn(1.0f, r) : 0.f;
    const float4* w4 = reinterpret_cast<const float4*>(ix.wL + (size_t)L * D);
    unsigned long long qp[kMaxM4][2];                 // q' as packed pairs (x, y), (z, w)
    float mn = INFINITY, mx = -INFINITY;
    const unsigned long long rinv2 = pk2(rinv, rinv);
#pragma unroll
    for (int m = 0; m < kMaxM4; ++m) {               // slots past D4 repeat slot D4 - 1 (min/max
      const int i = min(lane + 32 * m, D4 - 1);       // unchanged; their codes are not stored)
      const float4 w = __ldg(w4 + i), uu = u4[i];
      // q' = (u - w) / r   (r = 0: q' = 0), two elements per packed subtract and multiply
      qp[m][0] = mul_rn2(sub_rn2(pk2(uu.x, uu.y), pk2(w.x, w.y)), rinv2);
      qp[m][1] = mul_rn2(sub_rn2(pk2(uu.z, uu.w), pk2(w.z, w.w)), rinv2);
      const float2 a = up2(qp[m][0]), c = up2(qp[m][1]);
      mn = fminf(fminf(mn, a.x), a.y);
      mn = fminf(fminf(mn, c.x), c.y);
      mx = fmaxf(fmaxf(mx, a.x), a.y);
      mx = fmaxf(fmaxf(mx, c.x), c.y);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (!(r > 0.f)) mn = mx = 0.f;                    // q' = 0 exactly (no signed zeros)
    const float delta = __fdiv_rn(__fsub_rn(mx, mn), 15.0f);
    const float dinv = delta > 0.f ? __fdiv_rn(1.0f, delta) : 0.f;
    unsigned acc = 0;
    uint32_t* qrow = reinterpret_cast<uint32_t*>(qbar + (size_t)slot * D);   // row-major at the slot
    const unsigned long long mn2 = pk2(mn, mn), big2 = pk2(8388608.0f, 8388608.0f);
#pragma unroll
    for (int m = 0; m < kMaxM4; ++m) {
      const int i = lane + 32 * m;
      // t = fl(fl(q' - mn) * dinv) + 0.5 >= 0; clamp(floor(t), 0, 15) = floor(min(t, 15)), and
      // floor(t) = low bits of fl_down(t + 2^23) (spacing 1 in [2^23, 2^24)). dinv = 0: t = 0.5 -> 0.
      // The subtraction and the final round-down add two elements per packed instruction; the
      // multiply and + 0.5 stay scalar (ptxas contracts a packed mul.rn + add.rn pair into one
      // FFMA2, which would round once instead of twice).
      const float2 s01 = up2(sub_rn2(qp[m][0], mn2)), s23 = up2(sub_rn2(qp[m][1], mn2));
#define BBC_QT(x) fminf(__fadd_rn(__fmul_rn(x, dinv), 0.5f), 15.0f)
      const float2 g01 = up2(add_rm2(pk2(BBC_QT(s01.x), BBC_QT(s01.y)), big2));
      const float2 g23 = up2(add_rm2(pk2(BBC_QT(s23.x), BBC_QT(s23.y)), big2));
#undef BBC_QT
      const float f0 = g01.x, f1 = g01.y, f2 = g23.x, f3 = g23.y;
      const unsigned lo = __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x0040);
      const unsigned hi = __byte_perm(__float_as_uint(f2), __float_as_uint(f3), 0x0040);
      const unsigned v4 = __byte_perm(lo, hi, 0x5410);
      if (i < D4) qrow[i] = v4;
      acc = __dp4a(i < D4 ? v4 : 0u, 0x01010101u, acc);
    }
    int sq = (int)acc;
    sq = warp_sum(sq);
    if (lane == 0) {
      RbqPair e;
      e.c1 = __fdiv_rn(__fmul_rn(2.0f, delta), sD);
      e.c2 = __fdiv_rn(__fmul_rn(2.0f, mn), sD);
      e.c3 = __fsub_rn(-__fdiv_rn(__fmul_rn(delta, (float)sq), sD), __fmul_rn(sD, mn));
      e.r = r;
      e.rq2 = rq2;
      e.q = q;
      e.obase = (long long)q * b.cap + poff;
      pinfo[slot] = e;
    }
  }
}

// ------------------------------------------------------------------ pair layout
// Pairs estimated on the tensor cores: queries with a sample (nsamp > 0; otherwise tau = infinity
// and no estimate is needed) and lists non-empty on this shard.  The sample pass uses the pairs
// with j < nsamp, the Push pass all of them.  Slots: per list L, [off[L], off[L] + cnt_s[L]) the
// sample pairs, then the others up to off[L] + cnt_m[L]; off[L] is a multiple of kRbN.
__device__ __forceinline__ bool rbq_pair_sel(const Batch& b, const Dev& ix, long long p, int* L_out,
                                             bool* sample) {
  const int q = (int)(p / b.nprobe), j = (int)(p % b.nprobe);
  const int ns = b.nsamp[q];
  if (ns == 0) return false;
  const int L = b.probe[p];
  if (ix.loff[L + 1] == ix.loff[L]) return false;
  *L_out = L;
  *sample = j < ns;
  return true;
}

__global__ void k_rbq_lcount(Batch b, Dev ix, int* cnt_m, int* cnt_s) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)b.nq * b.nprobe) return;
  int L;
  bool smp;
  if (rbq_pair_sel(b, ix, p, &L, &smp)) {
    atomicAdd(&cnt_m[L], 1);
    if (smp) atomicAdd(&cnt_s[L], 1);
  }
}

__global__ void k_rbq_lfill(Batch b, Dev ix, int* cur_s, int* cur_m, int* islot) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)b.nq * b.nprobe) return;
  int L;
  bool smp;
  islot[p] = rbq_pair_sel(b, ix, p, &L, &smp) ? atomicAdd(smp ? &cur_s[L] : &cur_m[L], 1) : -1;
}

// off[L] = exclusive scan of cnt_m rounded up to kRbN; cur_s = off, cur_m = off + cnt_s (one CTA)
__global__ void __launch_bounds__(1024) k_rbq_lscan(const int* cnt_m, const int* cnt_s, int* off,
                                                    int* cur_s, int* cur_m, int nlist) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < nlist; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nlist ? (cnt_m[i] + kRbN - 1) / kRbN * kRbN : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int s = ws[lane];
      int y = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      ws[lane] = y - s;
    }
    __syncthreads();
    const int c0 = carry;
    if (i < nlist) {
      const int o = c0 + ws[wid] + x - v;
      off[i] = o;
      cur_s[i] = o;
      cur_m[i] = o + cnt_s[i];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + ws[wid] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[nlist] = carry;
}

// exclusive scan of cnt[nlist] -> off[nlist + 1]; cur = off (one CTA of 1024 threads)
__global__ void __launch_bounds__(1024) k_inv_scan(const int* cnt, int* off, int* cur, int nlist) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < nlist; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nlist ? cnt[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const int s = ws[lane];
      int y = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      ws[lane] = y - s;
    }
    __syncthreads();
    const int c0 = carry;
    if (i < nlist) {
      off[i] = c0 + ws[wid] + x - v;
      cur[i] = off[i];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + ws[wid] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[nlist] = carry;
}

// Per pair: the bucket-id function of its query's edges (after the sample stage), copied into
// the pair record so the GEMM epilogue reads it from shared memory with the other constants.
__global__ void k_rbq_paircell(Batch b, const int* __restrict__ islot, RbqPair* pinfo) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)b.nq * b.nprobe) return;
  const int slot = islot[p];
  if (slot < 0) return;
  const int q = (int)(p / b.nprobe);
  CellFn f;
  f.init(b.edges[2 * q], b.edges[2 * q + 1], b.nbuckets);
  RbqPair& e = pinfo[slot];
  e.dmin = f.dmin; e.dmax = f.dmax; e.inv = f.inv; e.bmax = f.bmax; e.degen = f.degen ? 1 : 0;
}

// Index-load-time: popcount of every code and the (list, 128-object tile) work list.
__global__ void k_rbq_popc(const uint8_t* bits, long long n, int D, int* pc) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(bits + r * (D / 8));
  int s = 0;
  for (int t = 0; t < D / 32; ++t) s += __popc(w[t]);
  pc[r] = s;
}

// ------------------------------------------------------------------ the list-major GEMM
struct RbqTc {
  const uint8_t* qbar;   // [slots x D] query codes, row-major (k_rbq_pairs; TMA tiles of kRbN rows)
  const RbqPair* pinfo;  // [slots]
  const int* off;        // [nlist + 1] first slot of each list (multiple of kRbN)
  const int* cnt_s;      // [nlist] sample pairs of each list
  const int* cnt_m;      // [nlist] all pairs of each list
  const int2* tiles;     // [ntiles] (list, first object)
  const int* pc;         // [n_local] popcount of each code
};

constexpr int kRbqIdesc = (2 << 4) | ((kRbN >> 3) << 17) | ((kRbM >> 4) << 24);   // s32 += u8 x u8

// A from tensor memory (lane = object row, 4 K bytes per 32-bit column), B from shared memory
__device__ __forceinline__ void i8_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"((uint32_t)kRbqIdesc), "r"(acc));
}

__device__ __forceinline__ uint32_t nib_bytes(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// ------------------------------------------------------------------ the list-major GEMM
// Warp-specialised pipeline.  Warp 24 (one lane) copies query tile qi -- kRbN slots of codes,
// row-major in global memory, by TMA into 128-byte-swizzled K blocks, plus their records by a bulk
// copy into ring entry qi % kRbRec -- into stage qi % nst; warp 25 (one lane) issues the MMAs of tile qi (A in tensor memory)
// into one of two TMEM accumulators; warps 0-23 run the epilogue of tile qi - 1 meanwhile (warp w
// reads TMEM lanes 32 (w & 3) .. +31 and pairs kPW (w >> 2) .. +kPW-1).  Measured: an MMA with
// N <= 64 costs ~51-57 cycles whatever N (tools/mma_microbench.cu), and the epilogue -- not the
// MMAs -- set the pace at N = 64 with 16 warps; N = 96 with 24 epilogue warps is faster.
// Hand-offs are mbarriers:
//   full[s]  (1 arrival + tx bytes)     tile landed in stage s
//   empty[s] (1 commit + 24 warps)      MMA read B and the epilogue read the records: stage free
//   accf[a]  (1 commit)                 accumulator a holds tile qi's products
//   acce[a]  (24 warps)                 accumulator a read out: free for tile qi + 2
constexpr int kRbWsEpi = 24, kRbWsNT = (kRbWsEpi + 2) * 32;   // 832 threads
constexpr int kRbRec = 4;                                      // records ring depth

template <bool SAMPLE>
__global__ void __launch_bounds__(kRbWsNT, 1) k_rbq_mma_ws(Batch b, Dev ix, RbqTc t, int nst,
                                                            const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) uint8_t rsm3[];
  const int D = ix.D;
  const int nkb = (D + 127) / 128;                                // 128-byte K blocks
  const int bst = nkb * kRbN * 128;                               // bytes per B stage
  uint8_t* sB = rsm3;                                             // [nst][nkb][32 x 128 B] swizzled
  RbqPair* pi = reinterpret_cast<RbqPair*>(sB + (size_t)nst * bst);   // [kRbRec][kRbN] records ring
  float* o_r = reinterpret_cast<float*>(pi + kRbRec * kRbN);      // [128] r_o
  float* o_g = o_r + kRbM;                                        // [128] 1 / g_o
  float* o_pc = o_g + kRbM;                                       // [128] popcount (float)
  // full[nst] empty[nst] (B stages: freed by the MMA commit alone) rfull[kRbRec] rempty[kRbRec]
  // (records: freed by the epilogue) accf[2] acce[2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(o_pc + kRbM);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * nst + 2 * kRbRec + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8u * nst;
  const uint32_t rfull0 = empty0 + 8u * nst, rempty0 = rfull0 + 8u * kRbRec;
  const uint32_t accf0 = rempty0 + 8u * kRbRec, acce0 = accf0 + 16u;

  const int2 tile = t.tiles[blockIdx.x];
  const int L = tile.x, o0 = tile.y;
  const int p0 = t.off[L], np = SAMPLE ? t.cnt_s[L] : t.cnt_m[L];
  if (np == 0) return;
  const long long row0 = ix.loff[L] + o0;
  const int nobj = min(kRbM, (int)(ix.loff[L + 1] - row0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = (np + kRbN - 1) / kRbN;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(full0 + 8u * i, 1);
      mbar_init(empty0 + 8u * i, 1);
    }
    for (int i = 0; i < kRbRec; ++i) {
      mbar_init(rfull0 + 8u * i, 1);
      mbar_init(rempty0 + 8u * i, kRbWsEpi);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(accf0 + 8u * a, 1);
      mbar_init(acce0 + 8u * a, kRbWsEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t rbytes = (uint32_t)(kRbN * sizeof(RbqPair));
  // copies of query tile qi into stage qi % nst (the first nst are issued before A is staged)
  auto load_tile = [&](int qi) {
    const int st = qi % nst, rs = qi % kRbRec;
    const uint32_t fb = full0 + 8u * st, rb = rfull0 + 8u * rs;
    mbar_arrive_tx(fb, (uint32_t)bst);
    mbar_arrive_tx(rb, rbytes);
    const int slot = p0 + qi * kRbN;
    const uint32_t dB = smem_u32(sB + (size_t)st * bst);
    for (int kb = 0; kb < nkb; ++kb) tma_2d_g2s(dB + kb * kRbN * 128, &tmB, 128 * kb, slot, fb);
    bulk_g2s(smem_u32(pi + rs * kRbN), t.pinfo + slot, rbytes, rb);
  };
  if (threadIdx.x == 0)
    for (int qi = 0; qi < min(nst, ntile); ++qi) load_tile(qi);
  __syncwarp();
  if (warp == 0) {                                    // all 512 columns: 2 accumulators + A
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tA = tmem + 2 * kRbN;                // A: columns [2 kRbN, 2 kRbN + D/4)
  // A: code bits of the tile's objects -> bytes 0/1 in tensor memory (lane = row); warp w of
  // 0-15 writes lanes 32 (w & 3) .. +31, 32-bit code words g = (w >> 2) + 4 i, 8 columns each
  if (warp < kRbWsEpi) {
    const int rq = warp & 3, r = 32 * rq + lane;
    const uint32_t* brow = reinterpret_cast<const uint32_t*>(ix.bits + (size_t)(row0 + min(r, nobj - 1)) * (D / 8));
    for (int g = warp >> 2; g < D / 32; g += kRbWsEpi / 4) {
      const uint32_t x = r < nobj ? brow[g] : 0u;
      const uint32_t taddr = tA + ((uint32_t)(32 * rq) << 16) + (uint32_t)(8 * g);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   ::"r"(taddr), "r"(nib_bytes(x & 15u)), "r"(nib_bytes((x >> 4) & 15u)),
                     "r"(nib_bytes((x >> 8) & 15u)), "r"(nib_bytes((x >> 12) & 15u)),
                     "r"(nib_bytes((x >> 16) & 15u)), "r"(nib_bytes((x >> 20) & 15u)),
                     "r"(nib_bytes((x >> 24) & 15u)), "r"(nib_bytes(x >> 28)) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (int r = threadIdx.x; r < kRbM; r += kRbWsNT) {
    float fr = 0.f, fg = 1.f, fp = 0.f;
    if (r < nobj) {
      const float2 f = reinterpret_cast<const float2*>(ix.factors)[row0 + r];
      fr = f.x; fg = __fdiv_rn(1.0f, f.y); fp = (float)t.pc[row0 + r];
    }
    o_r[r] = fr; o_g[r] = fg; o_pc[r] = fp;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (warp == kRbWsEpi) {
    // ---- producer: one lane; per query tile nkb TMA copies (kRbN rows x 128 B each) + one bulk
    // copy of the tile's kRbN records
    if (lane == 0) {
      for (int qi = nst; qi < ntile; ++qi) {
        mbar_wait(empty0 + 8u * (qi % nst), (unsigned)((qi / nst - 1) & 1));
        if (qi >= kRbRec) mbar_wait(rempty0 + 8u * (qi % kRbRec), (unsigned)((qi / kRbRec - 1) & 1));
        load_tile(qi);
      }
    }
    __syncwarp();
  } else if (warp == kRbWsEpi + 1) {
    // ---- MMA issuer
    if (lane == 0) {
      for (int qi = 0; qi < ntile; ++qi) {
        const int st = qi % nst, a = qi & 1;
        mbar_wait(full0 + 8u * st, (unsigned)((qi / nst) & 1));
        if (qi >= 2) mbar_wait(acce0 + 8u * a, (unsigned)((qi / 2 - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t d0 = umma_desc_sw128(smem_u32(sB + (size_t)st * bst));
        const uint32_t acc = tmem + (uint32_t)(a * kRbN);
        for (int k = 0; k < D / 32; ++k) {             // B start address advanced in 16-byte units
          const uint32_t oB = (uint32_t)(k >> 2) * (kRbN * 128u / 16u) + (uint32_t)(k & 3) * 2u;
          i8_mma_ts(acc, tA + (uint32_t)(8 * k), d0 + oB, k ? 1u : 0u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(accf0 + 8u * a) : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(empty0 + 8u * st) : "memory");
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: warps 0-23, thread = object row r, kPW pairs per warp
    constexpr int kPW = kRbN * 4 / kRbWsEpi;          // pairs per warp
    const int rq = warp & 3, cg = warp >> 2;
    const int r = 32 * rq + lane;
    float ro = 0.f, ginv = 0.f, pcf = 0.f;
    if (r < nobj) { ro = o_r[r]; ginv = o_g[r]; pcf = o_pc[r]; }
    const float a_ro = __fmul_rn(ro, ro), ro2 = __fmul_rn(2.0f, ro);
    for (int qi = 0; qi < ntile; ++qi) {
      const int a = qi & 1;
      const int nqt = min(kRbN, np - qi * kRbN);
      mbar_wait(accf0 + 8u * a, (unsigned)((qi / 2) & 1));
      const int rs = qi % kRbRec;
      mbar_wait(rfull0 + 8u * rs, (unsigned)((qi / kRbRec) & 1));   // records landed
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t v[kPW];
#pragma unroll
      for (int h = 0; h < kPW / 8; ++h) {
        const uint32_t taddr = tmem + ((uint32_t)(32 * rq) << 16) + (uint32_t)(a * kRbN + kPW * cg + 8 * h);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[8 * h + 0]), "=r"(v[8 * h + 1]), "=r"(v[8 * h + 2]), "=r"(v[8 * h + 3]),
                       "=r"(v[8 * h + 4]), "=r"(v[8 * h + 5]), "=r"(v[8 * h + 6]), "=r"(v[8 * h + 7])
                     : "r"(taddr));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acce0 + 8u * a);
      const RbqPair* P = pi + rs * kRbN;
      if (r < nobj) {
#pragma unroll
        for (int c = 0; c < kPW; ++c) {
          const int sp = kPW * cg + c;
          if (sp >= nqt) continue;
          const RbqPair& e = P[sp];
          const long long at = e.obase + o0 + r;
          // canonical estimator, identical to k_rbq_scan
          const float t1 = __fmul_rn(e.c2, pcf);
          const float t2 = __fadd_rn(t1, e.c3);
          // (float)v exactly, off the conversion pipe: 0 <= v < 2^23, so 2^23 + v is exact
          const float t3 = __fmul_rn(e.c1, __fsub_rn(__int_as_float((int)v[c] + 0x4B000000), 8388608.0f));
          const float oq = __fadd_rn(t3, t2);
          const float ee = __fmul_rn(oq, ginv);
          const float sum = __fadd_rn(a_ro, e.rq2);
          const float ff = __fmul_rn(ro2, e.r);
          const float est = __fsub_rn(sum, __fmul_rn(ff, ee));
          if (SAMPLE) {
            b.val[at] = est;
          } else {
            // bucket id (Eq. 6, R3), branch-free as CellFn: clamp(floor(x), 0, bmax) =
            // floor(clamp(x, 0, bmax)) (integer bounds; NaN -> 0), floor of y in [0, 255] = low
            // byte of fl_down(y + 2^23) -- no conversion-pipe instructions
            const float y = fminf(fmaxf(__fmul_rn(__fsub_rn(est, e.dmin), e.inv), 0.f), e.bmax);
            int cell = __float_as_int(__fadd_rd(y, 8388608.0f)) & 0xFF;
            cell = e.degen ? 0 : cell;
            cell = est > e.dmax ? 255 : cell;
            b.cells[at] = (uint8_t)cell;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(rempty0 + 8u * rs);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Histogram of the bucket ids < 255 of query q's probed objects (Push, Alg. 1 l.1-4).
__global__ void __launch_bounds__(256) k_cell_hist(Batch b) {
  __shared__ int h[8][kCells];
  const int q = blockIdx.y;
  if (b.nsamp[q] == 0) return;
  const int n = b.poff[(size_t)q * (b.nprobe + 1) + b.nprobe];
  const int wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * kCells; i += 256) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint8_t* c = b.cells + (size_t)q * b.cap;
  const int n16 = n >> 4;
  // plain shared atomics into per-warp copies (most ids are the uncounted 255: 16 of them are
  // skipped with one compare; warp aggregation by match measured slower on the PQ scans)
  // four 16-byte loads in flight per thread (the ids stream from DRAM once)
  const uint4* c16 = reinterpret_cast<const uint4*>(c);
  const int stride = gridDim.x * 256;
  for (int v0 = blockIdx.x * 256 + threadIdx.x; v0 < n16; v0 += 4 * stride) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      x[u] = v0 + u * stride < n16 ? c16[v0 + u * stride] : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((x[u].x & x[u].y & x[u].z & x[u].w) == 0xFFFFFFFFu) continue;
      const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int cell = (w[e >> 2] >> (8 * (e & 3))) & 255;
        if (cell < 255) atomicAdd(&h[wid][cell], 1);
      }
    }
  }
  if (blockIdx.x == 0)                               // ragged tail (< 16 objects)
    for (int i = (n16 << 4) + threadIdx.x; i < n; i += 256)
      if (c[i] < 255) atomicAdd(&h[wid][c[i]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < kCells; i += 256) {
    int t = 0;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) t += h[w8][i];
    if (t) atomicAdd(&b.hist[(size_t)q * kCells + i], t);
  }
}

}  // namespace bbc
