// a7, list-major exact re-rank with the rows staged in shared memory (BBC_RERANK_TILE).
//
// In list order (k_rerank_seg) every candidate row still travels L2 -> SM once per query that
// re-ranks it: each row of C4 is a candidate of ~19 queries of a micro-batch, and the kernel runs
// at ~0.8 of the L2 read bandwidth.  Here a CTA owns a tile of R consecutive rows of one inverted
// list: one bulk copy (cp.async.bulk, no per-row instructions) brings them from HBM into shared
// memory once, and the warps then compute every piece of that list -- (query, run of <= 64
// candidates) from k_rr_segments -- against the staged rows, reading them through the
// shared-memory pipe (128 B/clk/SM, ~2.4x the L2 -> SM rate).  Candidates of a piece outside the
// tile are left to the list's other tiles.  Per candidate the arithmetic is rr_rows32's (8 lanes
// per row, each lane's 16-byte chunks t = sl + 8v in order, fp32 FMAs, shuffle tree), so every
// distance is bit-identical to the query- and list-order kernels.  fp32 rows of <= 512 bytes.
#pragma once
#include "bbc_probe_tc.cuh"

namespace bbc {

constexpr int kRtNT = 512;                    // 16 warps
constexpr int kRtBytes = 96 * 1024;           // rows per tile = kRtBytes / row bytes (2 CTAs/SM)

__host__ __device__ constexpr int rt_rows(int rowb) { return kRtBytes / rowb; }

// Pieces per (list, tile) unit.  A segment -- the sorted run of candidate rows a query has in one
// list -- is cut at the list's tile boundaries (binary search of its rows) and each part into
// pieces of <= 64 candidates, counted (FILL = 0) or written (FILL = 1) at the unit's cursor, so
// every tile CTA sees exactly the candidates in its rows.  One thread per (query, probe) pair.
template <bool FILL>
__global__ void __launch_bounds__(256) k_rr_tile_pieces(Batch b, Dev ix, const int* __restrict__ ubase,
                                                        int* __restrict__ cnt, int4* __restrict__ seg) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (long long)b.nq * b.nprobe) return;
  const int2 g = rr_segment(b, p);
  if (g.y <= 0) return;
  const int q = (int)(p / b.nprobe);
  const int L = b.probe[p];
  const int R = rt_rows(ix.d * 4);
  const long long l0 = ix.loff[L];
  const int* cp = b.cpos + (size_t)q * b.cap + g.x;
  const int t0 = (int)((cp[0] - l0) / R), t1 = (int)((cp[g.y - 1] - l0) / R);
  int a = 0;
  for (int t = t0; t <= t1; ++t) {
    int e = g.y;                                     // first candidate of the segment past tile t
    if (t < t1) {
      const long long lim = l0 + (long long)(t + 1) * R;
      int lo = a, hi = g.y;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cp[mid] < lim) lo = mid + 1; else hi = mid;
      }
      e = lo;
    }
    const int n = e - a;
    if (n > 0) {
      const int np = (n + 63) / 64;
      const int at = atomicAdd(cnt + ubase[L] + t, np);
      if (FILL)
        for (int i = 0; i < np; ++i) seg[at + i] = make_int4(q, g.x + a + 64 * i, min(64, n - 64 * i), 0);
    }
    a = e;
  }
}

// ROWB = row bytes (384: C4, 512: C2).  A warp's 4 lane groups of 8 lanes work on 4 different
// pieces at once (each group holds its own query's slice in registers), so the dependent loads of
// a piece -- its record, candidate rows, ids, query -- of 4 pieces are in flight together; a group
// walks its piece's candidates in rounds of 8 (lane sl holds candidate 8i + sl's row and id).
template <int ROWB, bool IP>
__global__ void __launch_bounds__(kRtNT, 2) k_rerank_tile(Batch b, Dev ix, const int4* __restrict__ seg,
                                                          const int2* __restrict__ units,
                                                          const int* __restrict__ uoff) {
  constexpr int LPC = 8, NV = ROWB / 16, PER = (NV + LPC - 1) / LPC;
  constexpr int R = kRtBytes / ROWB;
  static_assert(NV % LPC == 0, "rows of whole 128-byte lane-group strides");
  extern __shared__ __align__(128) uint8_t rtsm[];
  __shared__ uint64_t bar;
  const int2 u = units[blockIdx.x];                   // (list, tile)
  const int L = u.x;
  const int p0 = uoff[blockIdx.x], p1 = uoff[blockIdx.x + 1];
  if (p0 == p1) return;                               // no candidate of this micro-batch in the tile
  const long long lo = ix.loff[L] + (long long)u.y * R;
  const long long hi = min(ix.loff[L + 1], lo + R);
  const uint32_t bsm = smem_u32(&bar);
  if (threadIdx.x == 0) {
    mbar_init(bsm, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)((hi - lo) * ROWB);
    mbar_arrive_tx(bsm, bytes);
    const uint8_t* src = static_cast<const uint8_t*>(ix.raw) + lo * ROWB;
    for (uint32_t o = 0; o < bytes; o += 32768u)
      bulk_g2s(smem_u32(rtsm) + o, src + o, min(32768u, bytes - o), bsm);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int grp = lane / LPC, sl = lane % LPC;
  const unsigned gmask = 0xFFu << (LPC * grp);
  const uint32_t tbase = smem_u32(rtsm) - (uint32_t)(lo * ROWB) + 16u * (uint32_t)sl;
  mbar_wait(bsm, 0);
#pragma unroll 1
  for (int pp = p0 + 4 * wid; pp < p1; pp += 4 * (kRtNT / 32)) {
    const int p = pp + grp;
    if (p >= p1) continue;                            // whole lane group idle
    const int4 pc = seg[p];                           // (query, first candidate, length <= 64)
    const int q = pc.x, n = pc.z;
    const size_t base = (size_t)q * b.cap + pc.y;
    float qr[PER][4];                                 // the lane's chunks t = sl + 8v of the query
    const float4* q4 = reinterpret_cast<const float4*>(b.Q + (size_t)q * ix.d);
#pragma unroll
    for (int v = 0; v < PER; ++v) {
      const float4 x = q4[sl + LPC * v];
      qr[v][0] = x.x; qr[v][1] = x.y; qr[v][2] = x.z; qr[v][3] = x.w;
    }
#pragma unroll 1
    for (int c0 = 0; c0 < n; c0 += LPC) {
      const int m = min(LPC, n - c0);
      const int rme = sl < m ? b.cpos[base + c0 + sl] : (int)lo;
      const int ime = sl < m ? (int)__ldg(ix.ids + rme) : 0;
#pragma unroll 1
      for (int c = 0; c < m; ++c) {
        const int rr = __shfl_sync(gmask, rme, c, LPC);
        const uint32_t row = tbase + (uint32_t)rr * (uint32_t)ROWB;
        float acc = 0.f;
#pragma unroll
        for (int v = 0; v < PER; ++v) {               // rr_rows32's order: chunk by chunk, x y z w
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(row + 16u * LPC * v));
          if (IP) {
            acc = fmaf(x.x, qr[v][0], acc);
            acc = fmaf(x.y, qr[v][1], acc);
            acc = fmaf(x.z, qr[v][2], acc);
            acc = fmaf(x.w, qr[v][3], acc);
          } else {
            const float a0 = x.x - qr[v][0], a1 = x.y - qr[v][1];
            const float a2 = x.z - qr[v][2], a3 = x.w - qr[v][3];
            acc = fmaf(a0, a0, acc);
            acc = fmaf(a1, a1, acc);
            acc = fmaf(a2, a2, acc);
            acc = fmaf(a3, a3, acc);
          }
        }
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o, LPC);
        if (sl == c) {                                // the lane holding this candidate's id writes
          b.val[base + c0 + c] = IP ? -acc : acc;
          b.cid[base + c0 + c] = ime;
        }
      }
    }
  }
}

}  // namespace bbc
