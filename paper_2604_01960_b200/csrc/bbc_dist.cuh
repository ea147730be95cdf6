// Kernels of the list-sharded (multi-GPU) query path.  DESIGN.md section 6.
//
// The database is partitioned by IVF list; every rank runs the steps of bbc_kernels.cuh on its
// own lists and the exchange steps below turn local counts into global decisions:
//   edges   d_min  = MIN over ranks of the local sample minimum               (all-reduce MIN)
//           d_max  = budget-th smallest sample estimate over all ranks: 4 radix passes of 8
//                    bits over the ordered 32-bit keys, each a 256-bin histogram (all-reduce SUM)
//   Push    the bucket histogram H (all-reduce SUM) -> one global threshold bucket tau
//   select  the k smallest (exact d^2, id) keys over all ranks' candidates: 8 radix passes
//           over 64-bit keys (all-reduce SUM of histograms); the per-(rank, query) counts of
//           selected pairs (all-reduce SUM); every rank packs its selected pairs query after
//           query and the packed runs are all-gathered (grouped broadcasts: an all-gather with
//           per-rank sizes) on a second stream and communicator, overlapping the next
//           micro-batch; each rank unpacks rank r's pairs of query q after those of ranks < r
// Integer sums and MIN are order independent, so the result is the same for every world size.
#pragma once
#include "bbc_kernels.cuh"

namespace bbc {

struct DistBuf {
  unsigned long long* prefix;  // [nq] radix prefix (bits above the current shift are decided)
  long long* need;             // [nq] rank of the wanted key among the undecided ones
  int* dh;                     // [nq x 256] pass histogram
  unsigned* umin;              // [nq] local/global minimum key
  int* tot;                    // [nq] global candidate count
  int* cnt;                    // [world x nq] selected candidates per rank
};

// ---------------------------------------------------------------- edges (32-bit value keys)
__global__ void __launch_bounds__(256) k_ds_edges_init(Batch b, DistBuf db) {
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q >= b.nq) return;
  db.prefix[q] = 0;
  db.need[q] = b.nsamp[q] > 0 ? b.budget : 0;
}

// local minimum of the sample estimates (0xffffffff when this rank holds none)
__global__ void __launch_bounds__(256) k_ds_localmin(Batch b, DistBuf db) {
  __shared__ unsigned red[8];
  const int q = blockIdx.x;
  const int ns = b.nsamp[q];
  const int n = ns > 0 ? b.poff[(size_t)q * (b.nprobe + 1) + ns] : 0;
  const float* v = b.val + (size_t)q * b.cap;
  unsigned m = 0xffffffffu;
  for (int i = threadIdx.x; i < n; i += 256) m = min(m, f2key(v[i]));
  m = warp_min(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned r = red[0];
    for (int w = 1; w < 8; ++w) r = min(r, red[w]);
    db.umin[q] = r;
  }
}

// histogram of digit (key >> shift) & 255 over the local keys that match the decided prefix
template <bool FINAL>
__global__ void __launch_bounds__(256) k_ds_hist(Batch b, DistBuf db, int shift) {
  __shared__ int h[kCells];
  const int q = blockIdx.y;
  if (db.need[q] <= 0) return;
  int n;
  if (FINAL) {
    n = b.ncand[q];
  } else {
    const int ns = b.nsamp[q];
    n = ns > 0 ? b.poff[(size_t)q * (b.nprobe + 1) + ns] : 0;
  }
  if (blockIdx.x * 256 >= n) return;
  for (int i = threadIdx.x; i < kCells; i += 256) h[i] = 0;
  __syncthreads();
  const unsigned long long pref = db.prefix[q];
  const float* v = b.val + (size_t)q * b.cap;
  const int* id = b.cid + (size_t)q * b.cap;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    const unsigned long long key =
        FINAL ? (((unsigned long long)f2key(v[i]) << 32) | (unsigned)id[i]) : (unsigned long long)f2key(v[i]);
    if (shr64(key, shift + 8) == shr64(pref, shift + 8)) atomicAdd(&h[(key >> shift) & 255u], 1);
  }
  __syncthreads();
  int* g = db.dh + (size_t)q * kCells;
  for (int i = threadIdx.x; i < kCells; i += 256)
    if (h[i]) atomicAdd(&g[i], h[i]);
}

// pick the digit holding the need-th key (global histogram; identical on every rank)
__global__ void __launch_bounds__(32) k_ds_pick(Batch b, DistBuf db, int shift) {
  const int q = blockIdx.x, lane = threadIdx.x;
  const long long need = db.need[q];
  if (need <= 0) return;
  const int* H = db.dh + (size_t)q * kCells;
  long long v[8], s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = H[lane * 8 + j]; s += v[j]; }
  long long incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  long long c = incl - s;
  if (c < need && need <= incl) {
    for (int j = 0; j < 8; ++j) {
      if (c + v[j] >= need) {
        db.prefix[q] |= (unsigned long long)(lane * 8 + j) << shift;
        db.need[q] = need - c;
        break;
      }
      c += v[j];
    }
  }
}

__global__ void __launch_bounds__(256) k_ds_edges_finish(Batch b, DistBuf db) {
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q >= b.nq || b.nsamp[q] == 0) return;
  b.edges[2 * q] = key2f(db.umin[q]);
  b.edges[2 * q + 1] = key2f((unsigned)db.prefix[q]);
  atomicAdd((unsigned long long*)&b.stats[2],
            (unsigned long long)b.poff[(size_t)q * (b.nprobe + 1) + b.nsamp[q]]);
}

// ---------------------------------------------------------------- final selection (64-bit keys)
__global__ void __launch_bounds__(256) k_ds_final_init(Batch b, DistBuf db) {
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q >= b.nq) return;
  const int t = db.tot[q];                 // global |S*|
  db.prefix[q] = t > b.k ? 0ull : ~0ull;   // ~0: every candidate is selected
  db.need[q] = t > b.k ? b.k : 0;
}

__global__ void __launch_bounds__(256) k_ds_ncand(Batch b, DistBuf db) {
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q < b.nq) db.tot[q] = b.ncand[q];
}

// The result exchange buffers of one micro-batch (fixed offsets in the workspace, sized for the
// largest micro-batch): this rank's packed selected pairs, every rank's packed pairs after the
// all-gather, and the per-(rank, query) counts and packed offsets the unpack needs.
struct XBuf {
  unsigned long long* send;    // [nqmax x k]  (fp32 bits of d^2) << 32 | id, query after query
  unsigned long long* recv;    // [nqmax x k]  rank r's run at displs[r]
  int* cnt;                    // [world x nqmax] selected pairs of (rank, query)
  int* coff;                   // [world x nqmax] offset of (rank, query) in rank's packed run
  long long* tot;              // [world] pairs packed by each rank
};
struct Displs {
  long long d[8];              // first element of rank r's run in recv (world <= 8)
};

// count (FILL=false) or pack (FILL=true: in candidate order at send[coff[rank][q]]) the local
// candidates whose key is <= the selected threshold
template <bool FILL>
__global__ void __launch_bounds__(kSelNT) k_ds_select(Batch b, DistBuf db, int rank, XBuf xb) {
  __shared__ int wcnt[kSelNT / 32 + 1];
  const int q = blockIdx.x;
  const int nc = b.ncand[q];
  const unsigned long long thr = db.prefix[q];
  const float* v = b.val + (size_t)q * b.cap;
  const int* id = b.cid + (size_t)q * b.cap;
  unsigned long long* out = FILL ? xb.send + xb.coff[(size_t)rank * b.nq + q] : nullptr;
  const int mine = FILL ? xb.cnt[(size_t)rank * b.nq + q] : 0;
  int base = 0;
  for (int t0 = 0; t0 < nc; t0 += kSelNT) {
    const int i = t0 + threadIdx.x;
    bool f = false;
    unsigned long long key = 0;
    if (i < nc) {
      key = ((unsigned long long)f2key(v[i]) << 32) | (unsigned)id[i];
      f = key <= thr;
    }
    int total;
    const int r = block_rank<kSelNT>(f, wcnt, &total);
    if (FILL && f && base + r < mine)
      out[base + r] = ((unsigned long long)__float_as_uint(v[i]) << 32) | (unsigned)id[i];
    base += total;
  }
  if (!FILL && threadIdx.x == 0) db.cnt[(size_t)rank * b.nq + q] = base;
}

// Per rank r (one CTA each): the counts of the micro-batch's queries copied into the exchange
// buffer, their exclusive scan over queries (packed offsets) and the total.
__global__ void __launch_bounds__(1024) k_ds_counts_scan(Batch b, DistBuf db, XBuf xb) {
  __shared__ int ws[32];
  __shared__ long long carry;
  const int r = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < b.nq; base += 1024) {
    const int q = base + threadIdx.x;
    const int v = q < b.nq ? db.cnt[(size_t)r * b.nq + q] : 0;
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
    const long long c0 = carry;
    if (q < b.nq) {
      xb.cnt[(size_t)r * b.nq + q] = v;
      xb.coff[(size_t)r * b.nq + q] = (int)(c0 + ws[wid] + x - v);
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + ws[wid] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) xb.tot[r] = carry;
}

// After the all-gather: row q = rank 0's pairs of q, then rank 1's, ...; padding (-1, +inf) past
// the global count.  One CTA per query.
__global__ void __launch_bounds__(256) k_ds_unpack(int nq, int k, int world, XBuf xb, Displs dp,
                                                   long long* out_ids, float* out_d2) {
  const int q = blockIdx.x;
  long long* oi = out_ids + (size_t)q * k;
  float* od = out_d2 + (size_t)q * k;
  int base = 0;
  for (int r = 0; r < world; ++r) {
    const int c = min(xb.cnt[(size_t)r * nq + q], k - base);
    const unsigned long long* src = xb.recv + dp.d[r] + xb.coff[(size_t)r * nq + q];
    for (int i = threadIdx.x; i < c; i += 256) {
      const unsigned long long x = src[i];
      oi[base + i] = (long long)(unsigned)(x & 0xffffffffull);
      od[base + i] = __uint_as_float((unsigned)(x >> 32));
    }
    base += c;
  }
  for (int i = base + threadIdx.x; i < k; i += 256) {
    oi[i] = -1;
    od[i] = INFINITY;
  }
}

// ---------------------------------------------------------------- local-group reduction
// Single-process group of G shards on one device: element-wise reduction of G buffers, written
// back to all of them (all-reduce semantics).  op 0 = sum, 1 = min.
struct GroupPtrs {
  void* p[8];
};
template <typename T>
__global__ void k_group_allreduce(GroupPtrs ptrs, int G, long long n, int op) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    T r = static_cast<T*>(ptrs.p[0])[i];
    for (int g = 1; g < G; ++g) {
      const T v = static_cast<T*>(ptrs.p[g])[i];
      r = op == 0 ? (T)(r + v) : (v < r ? v : r);
    }
    for (int g = 0; g < G; ++g) static_cast<T*>(ptrs.p[g])[i] = r;
  }
}

}  // namespace bbc
