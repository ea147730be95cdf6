// Kernels of the list-sharded (multi-GPU) query path.  DESIGN.md section 6.
//
// The database is partitioned by IVF list; every rank runs the steps of bbc_kernels.cuh on its
// own lists and the exchange steps below turn local counts into global decisions:
//   edges   d_min  = MIN over ranks of the local sample minimum               (all-reduce MIN)
//           d_max  = budget-th smallest sample estimate over all ranks: 4 radix passes of 8
//                    bits over the ordered 32-bit keys, each a 256-bin histogram (all-reduce SUM)
//   Push    the bucket histogram H (all-reduce SUM) -> one global threshold bucket tau
//   select  the k smallest (exact d^2, id) keys over all ranks' candidates: 8 radix passes
//           over 64-bit keys (all-reduce SUM of histograms), then every rank writes its
//           selected pairs at its offset of a zeroed output that is summed across ranks
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

// count (FILL=false) or write (FILL=true, in candidate order, at this rank's offset) the local
// candidates whose key is <= the selected threshold
template <bool FILL>
__global__ void __launch_bounds__(kSelNT) k_ds_select(Batch b, DistBuf db, int rank, int world,
                                                      long long* out_ids, float* out_d2) {
  __shared__ int wcnt[kSelNT / 32 + 1];
  const int q = blockIdx.x;
  const int nc = b.ncand[q];
  const unsigned long long thr = db.prefix[q];
  const float* v = b.val + (size_t)q * b.cap;
  const int* id = b.cid + (size_t)q * b.cap;
  int off = 0;
  if (FILL)
    for (int r = 0; r < rank; ++r) off += db.cnt[(size_t)r * b.nq + q];
  int base = 0;
  for (int t0 = 0; t0 < nc; t0 += kSelNT) {
    const int i = t0 + threadIdx.x;
    bool f = false;
    if (i < nc) f = ((((unsigned long long)f2key(v[i]) << 32) | (unsigned)id[i]) <= thr);
    int total;
    const int r = block_rank<kSelNT>(f, wcnt, &total);
    if (FILL && f && off + base + r < b.k) {
      out_ids[(size_t)q * b.k + off + base + r] = id[i];
      out_d2[(size_t)q * b.k + off + base + r] = v[i];
    }
    base += total;
  }
  if (!FILL && threadIdx.x == 0) db.cnt[(size_t)rank * b.nq + q] = base;
}

// after the output sum: positions past the global count are padding
__global__ void __launch_bounds__(256) k_ds_pad(Batch b, DistBuf db, int world, long long* out_ids,
                                                float* out_d2) {
  const int q = blockIdx.y;
  int n = 0;
  for (int r = 0; r < world; ++r) n += db.cnt[(size_t)r * b.nq + q];
  for (int i = n + blockIdx.x * 256 + threadIdx.x; i < b.k; i += gridDim.x * 256) {
    out_ids[(size_t)q * b.k + i] = -1;
    out_d2[(size_t)q * b.k + i] = INFINITY;
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
