// Host side of libbbc.so: index loading (ivf_load), workspace planning, and the launch sequence
// of the query path (bbc_search).  C ABI declared in include/bbc.h.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "bbc.h"
#include <nccl.h>

#include "bbc_dist.cuh"
#include "bbc_probe_tc.cuh"
#include "bbc_rbq_tc.cuh"
#include "bbc_pq4.cuh"
#include "bbc_rerank_tile.cuh"
#include "bbc_alg3.cuh"

using namespace bbc;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

bbc_status fail(bbc_status s, const std::string& m) {
  g_err = m;
  return s;
}

struct Timer {
  int stage;
  cudaEvent_t a, b;
};

}  // namespace

struct bbc_index_s {
  int device = 0;
  int rank = 0, world = 1;
  int kind = 0, d = 0, nlist = 0, M = 0, D = 0, raw_u8 = 0, metric = BBC_METRIC_L2;
  int nbits = 8;                        // PQ code bits: 8 (replicated-LUT scan) or 4 (bbc_pq4.cuh)
  long long N = 0, n_local = 0;
  int max_list = 0;
  std::vector<int> lsize;               // local list sizes
  std::vector<int> gsize;               // global list sizes
  std::vector<long long> desc_prefix;   // prefix sums of local sizes sorted descending
  // device arrays
  float* centroids = nullptr;
  long long* loff = nullptr;
  int* gsize_d = nullptr;
  long long* ids = nullptr;
  float* books = nullptr;
  uint8_t* codes = nullptr;
  float* P = nullptr;
  float* wL = nullptr;
  uint8_t* bits = nullptr;
  float* factors = nullptr;
  void* raw = nullptr;
  long long* stats = nullptr;           // [kNStats]
  uint8_t* codes_t = nullptr;           // PQ codes, per-list chunk-major (8-bit: replicated-LUT scan;
                                        // 4-bit: k_pack_codes4 layout)
  long long* tbase = nullptr;           // [nlist] byte offset of each list in codes_t
  long long ct_bytes = 0;               // bytes of codes_t (without the tail pad)
  float* cmu = nullptr;                 // [d] centroid mean (tensor-core probe)
  float* pb_hi = nullptr;               // [nlist_pad x d] centred centroids, tf32 hi part (d <= 128)
  float* pb_lo = nullptr;               //                 and the remainder
  CUtensorMap ptm_hi, ptm_lo;           // their TMA maps (k_probe_mma_ws)
  bool probe_ws_ok = false;
  float* cnorm = nullptr;               // [nlist] |c - mu|^2
  int* lrank = nullptr;                 // [nlist] (region << 20 | list): query locality order
  float cmax = 0.f;                     // max |c - mu|, rounded up
  int probe_mode = BBC_PROBE_AUTO;       // BBC_PROBE_* (bbc_probe_tc.cuh)
  int nbuckets = 255;                   // B regular buckets of the result buffer (Eq. 6)
  bool probe_tc_ok = false;             // d <= 1024: the tensor-core probe is available
  int rbq_tc = 0;                       // 1: RaBitQ estimates on the tensor cores (bbc_rbq_tc.cuh)
  int rerank_order = BBC_RERANK_AUTO;    // BBC_RERANK_*: work order of the exact re-rank (a7)
  int remap_m = 0;                       // 0 or m equal-depth buckets (bbc_set_remap)
  int alg3 = 0;                          // 1: Algorithm 3 bound-aware re-rank (bbc_set_bound_rerank)
  int early = 0;                         // 1: Algorithm 4 early re-ranking of IVF+PQ (bbc_set_early_rerank)
  float alg3_eps0 = 1.9f;                // its bound's eps0
  int code_loads = BBC_CODES_AUTO;       // BBC_CODES_*: L1 policy of the PQ scan's code loads
  int scan_order = BBC_ORDER_AUTO;        // BBC_SCAN_*: visiting order of the 8-bit PQ scan
  int2* rt_units = nullptr;             // [rt_nunits] (list, tile) of the shared-memory re-rank
  int rt_nunits = 0;                    //   (BBC_RERANK_TILE; fp32 rows of <= 512 bytes)
  int* rt_ubase = nullptr;              // [nlist] first unit of each list
  int rt_maxtiles = 0;                  // most tiles of one list
  int2* rbq_tiles = nullptr;            // [rbq_ntiles] (list, first object) of 128-object tiles
  int rbq_ntiles = 0;
  int* rbq_pc = nullptr;                // [n_local] popcount of each code
  bool broken = false;
  bool timing = false;
  std::vector<Timer> timers;
  std::vector<cudaEvent_t> pool;
  double stage_ms[BBC_NUM_STAGES] = {0};
  long long timed_calls = 0;
  long long microbatches = 0;
  long long rr_list_batches = 0;        // micro-batches of the last search re-ranked in list order
  int num_sms = 148;
  int l2_bytes = 126 << 20;
  void* nccl = nullptr;                 // ncclComm_t of this rank (bbc_comm_init)
  long long* nccl_scratch = nullptr;    // [1] device scalar of the host-value agreement
  void* nccl_x = nullptr;               // ncclComm_t split from nccl: the result all-gather on the
                                        // copy stream, concurrent with the next micro-batch's collectives
  long long* h_tot = nullptr;           // [8] pinned host: pairs each rank packs (exchange sizes)
  int force_dist = 0;                   // run the sharded code path even at world 1 (tests)
  cudaStream_t copy_stream = nullptr;   // host path: device->host result copies
  cudaStream_t copy_stream2 = nullptr;  //   (the distances on a second copy stream and engine)
  cudaEvent_t ev_copied2[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
};

namespace {

#define CU(expr)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      if (ix) ix->broken = true;                                                   \
      return fail(BBC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    }                                                                              \
  } while (0)

#define CU_NOIX(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) return fail(BBC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

Dev dev_view(const bbc_index_s* ix) {
  Dev v;
  v.kind = ix->kind; v.d = ix->d; v.nlist = ix->nlist; v.M = ix->M; v.D = ix->D;
  v.ksub = 1 << ix->nbits;
  v.raw_u8 = ix->raw_u8; v.n_local = ix->n_local; v.metric = ix->metric;
  v.centroids = ix->centroids; v.loff = ix->loff; v.gsize = ix->gsize_d; v.ids = ix->ids;
  v.books = ix->books; v.codes = ix->codes; v.P = ix->P; v.wL = ix->wL; v.bits = ix->bits;
  v.factors = ix->factors; v.raw = ix->raw;
  v.cmu = ix->cmu; v.cnorm = ix->cnorm; v.cmax = ix->cmax; v.probe_tc = 0;
  v.ct_bytes = ix->ct_bytes;
  return v;
}

cudaEvent_t take_event(bbc_index_s* ix) {
  if (!ix->pool.empty()) {
    cudaEvent_t e = ix->pool.back();
    ix->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct StageScope {
  bbc_index_s* ix;
  cudaStream_t st;
  Timer t;
  bool on;
  StageScope(bbc_index_s* i, cudaStream_t s, int stage) : ix(i), st(s), on(i->timing) {
    if (on) {
      t.stage = stage;
      t.a = take_event(ix);
      t.b = take_event(ix);
      cudaEventRecord(t.a, st);
    }
  }
  ~StageScope() {
    if (on) {
      cudaEventRecord(t.b, st);
      ix->timers.push_back(t);
    }
  }
};

struct RbqBufs {
  uint8_t* qbar = nullptr;     // [slots x D] query codes, row-major (TMA loads kRbN-slot tiles)
  RbqPair* pinfo = nullptr;    // [slots]
  int* islot = nullptr;        // [nq x nprobe] slot of each pair (-1: not estimated)
  int* cnt_m = nullptr;        // [nlist + 1] pairs per list
  int* cnt_s = nullptr;        // [nlist + 1] sample pairs per list
  int* off = nullptr;          // [nlist + 1] first slot per list (multiple of kRbN)
  int* cur_s = nullptr;        // [nlist + 1] fill cursors
  int* cur_m = nullptr;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int kItemMin = kRqE < kQ4Item ? kRqE : kQ4Item;   // smallest scan work item (sizes the item list)

struct Plan {
  long long cap;      // per-query element capacity
  size_t per_query;   // bytes per query
  size_t fixed;       // alignment slack
};

// world: ranks of the exchange (>= 1); xchg: the sharded path runs (its result-exchange buffers
// are needed even with a 1-rank communicator)
Plan make_plan(const bbc_index_s* ix, int nprobe, int k, int world = 1, bool xchg = false) {
  Plan p;
  long long cap = ix->desc_prefix[std::min<size_t>(nprobe, ix->desc_prefix.size() - 1)];
  cap = (cap + 15) / 16 * 16;
  if (cap < 16) cap = 16;
  p.cap = cap;
  size_t table = ix->kind == BBC_KIND_PQ ? (size_t)ix->M * 256 * 4 : (size_t)ix->D * 4;
  p.per_query = (size_t)ix->nlist * 4 + (size_t)nprobe * 20 + 8 +
                (size_t)((cap + 32LL * nprobe + kItemMin - 1) / kItemMin) * 8 + 4 + 8 + kCells * 4 + 4 + 4 +
                table + (size_t)cap * 13 + (size_t)ix->d * 4 + (size_t)k * 24 + 64 +
                (size_t)((cap + kChunk - 1) / kChunk) * 8 + (size_t)(nprobe + 1) * 4;
  p.per_query += 8 + 8 + kCells * 4 + 4 + 4 + (size_t)4 * world;   // DistBuf
  const int piece = rr_piece(ix->raw_u8 ? ix->d : 4 * ix->d);
  p.per_query += (size_t)nprobe * 20 + (size_t)(cap / piece) * 16;      // re-rank pieces
  p.per_query += (size_t)nprobe * ix->rt_maxtiles * 16;                   //   + cuts at tile bounds
  p.per_query += kCells + 4;                                             // remap, nest
  p.per_query += (size_t)(2 * nprobe + 1) * 4 +                          // sweep order (sperm, spad)
                 (size_t)((cap + 32LL * nprobe + kItemMin - 1) / kItemMin) * 12;   //   + items_s, ikey
  if (xchg || world > 1) p.per_query += (size_t)k * 16 + (size_t)world * 8;   // result exchange (XBuf)
  if (ix->alg3) p.per_query += (size_t)cap * 12 + 8 + 4 * 256;          // Algorithm 3 (a3lb, a3lc, a3ordu, a3pos)
  if (ix->early) p.per_query += (size_t)cap * 4 + 4 + 2 * 256;          // Algorithm 4 (early, tpred)
  p.fixed = 64 * 256 + (size_t)3 * (std::max(ix->nlist, ix->rt_nunits) + 1) * 4 + 3 * 256 +
            (size_t)(ix->nlist + 1) * 4 + 512;                          // icnt, ictr
  if (ix->kind == BBC_KIND_RABITQ && ix->rbq_tc) {            // pair codes + inverted index
    p.per_query += (size_t)nprobe * ((size_t)ix->D + sizeof(RbqPair) + 4);   // codes, records, slots
    p.fixed += (size_t)kRbN * ix->nlist * ((size_t)ix->D + sizeof(RbqPair)) +   // per-list padding
               (size_t)5 * (ix->nlist + 1) * 4 + 8 * 256;
  }
  return p;
}

// Carve the micro-batch arrays out of the workspace.  The query and output staging buffers come
// first, sized for the largest micro-batch (nqmax), so they sit at the same offsets in every
// micro-batch of a search: the host path's device->host copy of micro-batch i (copy stream) may
// still read its output buffer while micro-batch i+1 (possibly smaller: the tail halves) runs.
void carve(const bbc_index_s* ix, const Plan& p, int nqb, int nqmax, int nprobe, char* ws, Batch& b,
           float** qstage, long long** ostage_ids, float** ostage_d2, int k, DistBuf* db, int world,
           RbqBufs* rb, XBuf* xb) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = ws + off;
    off = align256(off + bytes);
    return r;
  };
  *qstage = (float*)take((size_t)nqmax * ix->d * 4);
  *ostage_ids = (long long*)take((size_t)nqmax * k * 8);
  *ostage_d2 = (float*)take((size_t)nqmax * k * 4);
  b.ostage2_ids = (long long*)take((size_t)nqmax * k * 8);   // second output staging (host path)
  b.ostage2_d2 = (float*)take((size_t)nqmax * k * 4);
  if (xb) {                         // result exchange: read by the copy stream past this micro-batch
    xb->send = (unsigned long long*)take((size_t)nqmax * k * 8);
    xb->recv = (unsigned long long*)take((size_t)nqmax * k * 8);
    xb->cnt = (int*)take((size_t)world * nqmax * 4);
    xb->coff = (int*)take((size_t)world * nqmax * 4);
    xb->tot = (long long*)take((size_t)world * 8);
  }
  size_t table = ix->kind == BBC_KIND_PQ ? (size_t)ix->M * 256 : (size_t)ix->D;
  b.coarse = (float*)take((size_t)nqb * ix->nlist * 4);
  b.probe = (int*)take((size_t)nqb * nprobe * 4);
  b.rq2 = (float*)take((size_t)nqb * nprobe * 4);
  b.poff = (int*)take((size_t)nqb * (nprobe + 1) * 4);
  b.popad = (int*)take((size_t)nqb * (nprobe + 1) * 4);
  b.rbase = (long long*)take((size_t)nqb * nprobe * 8);
  b.qperm = (int*)take((size_t)nqb * 4);
  b.items = (int2*)take((size_t)nqb * ((p.cap + 32LL * nprobe + kItemMin - 1) / kItemMin) * 8);
  b.nitems = (int*)take(4);
  b.sperm = (int*)take((size_t)nqb * nprobe * 4);
  b.spad = (int*)take((size_t)nqb * (nprobe + 1) * 4);
  b.items_s = (int2*)take((size_t)nqb * ((p.cap + 32LL * nprobe + kItemMin - 1) / kItemMin) * 8);
  b.ikey = (int*)take((size_t)nqb * ((p.cap + 32LL * nprobe + kItemMin - 1) / kItemMin) * 4);
  b.icnt = (int*)take((size_t)(ix->nlist + 1) * 4);
  b.nsamp = (int*)take((size_t)nqb * 4);
  // with the sweep order (codes streamed from HBM), the 8-bit PQ scan's sample pass fills its
  // last work item with the following lists (C4 103.4 vs 104.3 ms per step; L2-resident C2,
  // whose sample pass skips the idle warps of its last item, 5.00 vs 4.96 ms: not there)
  const bool pq8 = ix->kind == BBC_KIND_PQ && ix->nbits == 8 &&
                   (ix->scan_order == BBC_ORDER_SWEEP ||
                    (ix->scan_order == BBC_ORDER_AUTO && (double)ix->n_local * ix->M > 0.5 * (double)ix->l2_bytes));
  b.nest = pq8 ? (int*)take((size_t)nqb * 4) : b.nsamp;
  b.nest_item = pq8 ? kRqE : 0;
  b.edges = (float*)take((size_t)nqb * 8);
  b.hist = (int*)take((size_t)nqb * kCells * 4);
  b.tau = (int*)take((size_t)nqb * 4);
  b.ncand = (int*)take((size_t)nqb * 4);
  b.table = (float*)take((size_t)nqb * table * 4);
  b.cells = (uint8_t*)take((size_t)nqb * p.cap);
  b.cpos = (int*)take((size_t)nqb * p.cap * 4);
  b.cid = (int*)take((size_t)nqb * p.cap * 4);
  b.val = (float*)take((size_t)nqb * p.cap * 4);
  b.chunk = (int*)take((size_t)nqb * ((p.cap + kChunk - 1) / kChunk) * 4);
  b.chunkj = (int*)take((size_t)nqb * ((p.cap + kChunk - 1) / kChunk) * 4);
  b.sstart = (int*)take((size_t)nqb * nprobe * 4);
  b.rmap = (uint8_t*)take((size_t)nqb * kCells);
  b.rseg = (int4*)take((size_t)nqb * ((size_t)nprobe * (1 + ix->rt_maxtiles) +
                                       p.cap / rr_piece(ix->raw_u8 ? ix->d : 4 * ix->d)) * 16);
  const size_t nrs = (size_t)std::max(ix->nlist, ix->rt_nunits) + 1;   // lists, or tile units
  b.rs_cnt = (int*)take(nrs * 4);
  b.rs_off = (int*)take(nrs * 4);
  b.rs_cur = (int*)take(nrs * 4);

  if (ix->alg3) {
    b.a3lb = (uint16_t*)take((size_t)nqb * p.cap * 2);
    b.a3lc = (uint16_t*)take((size_t)nqb * p.cap * 2);
    b.a3ordu = (int*)take((size_t)nqb * p.cap * 4);
    b.a3nall = (int*)take((size_t)nqb * 4);
    b.a3pos = ix->alg3 == BBC_ALG3_LIST ? (int*)take((size_t)nqb * p.cap * 4) : nullptr;
    b.a3tau = (int*)take((size_t)nqb * 4);
  } else {
    b.a3lb = b.a3lc = nullptr;
    b.a3ordu = b.a3nall = b.a3pos = b.a3tau = nullptr;
  }
  if (ix->early) {
    b.early = (float*)take((size_t)nqb * p.cap * 4);
    b.tpred = (int*)take((size_t)nqb * 4);
  } else {
    b.early = nullptr;
    b.tpred = nullptr;
  }
  db->prefix = (unsigned long long*)take((size_t)nqb * 8);
  db->need = (long long*)take((size_t)nqb * 8);
  db->dh = (int*)take((size_t)nqb * kCells * 4);
  db->umin = (unsigned*)take((size_t)nqb * 4);
  db->tot = (int*)take((size_t)nqb * 4);
  db->cnt = (int*)take((size_t)nqb * world * 4);
  if (ix->kind == BBC_KIND_RABITQ && ix->rbq_tc) {
    const size_t pairs = (size_t)nqb * nprobe;
    const size_t slots = pairs + (size_t)kRbN * ix->nlist;   // each list padded to kRbN slots
    rb->qbar = (uint8_t*)take(slots * ix->D);
    rb->pinfo = (RbqPair*)take(slots * sizeof(RbqPair));
    rb->islot = (int*)take(pairs * 4);
    rb->cnt_m = (int*)take((size_t)(ix->nlist + 1) * 4);
    rb->cnt_s = (int*)take((size_t)(ix->nlist + 1) * 4);
    rb->off = (int*)take((size_t)(ix->nlist + 1) * 4);
    rb->cur_s = (int*)take((size_t)(ix->nlist + 1) * 4);
    rb->cur_m = (int*)take((size_t)(ix->nlist + 1) * 4);
  }
}

template <typename Kern>
void set_smem(Kern kern, size_t bytes) {
  if (bytes > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

__global__ void k_iota(int* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

__global__ void k_debug_cands(const int* cpos, const float* val, const int* ncand, long long cap,
                              long long* out_ids, float* out_d2, long long stride,
                              const int* rows = nullptr, uint8_t* out_early = nullptr) {
  const int q = blockIdx.y;
  const int n = ncand[q];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n && i < stride;
       i += (long long)gridDim.x * blockDim.x) {
    if (out_ids) out_ids[q * stride + i] = cpos[q * cap + i];
    if (out_d2) out_d2[q * stride + i] = val[q * cap + i];
    if (out_early) out_early[q * stride + i] = rows && rows[q * cap + i] < 0;   // Algorithm 4
  }
}

template <int M>
void launch_rq(bool est, int grid, cudaStream_t st, const Batch& b, const Dev& dv,
               const uint8_t* ct, const long long* tb, float* out, long long stride, int mode, bool na,
               bool sweep) {
#define BBC_RQ_L(E, NA)                                                                                  \
  do {                                                                                                  \
    set_smem(k_pq_scan_rq<M, E, NA>, kRqSmem);                                                          \
    k_pq_scan_rq<M, E, NA><<<grid, kRqNT, kRqSmem, st>>>(b, dv, ct, tb, out, stride, mode,              \
                                                          sweep ? b.items_s : b.items, b.nitems,        \
                                                          sweep ? b.sperm : nullptr);                   \
  } while (0)
  if (est) { if (na) BBC_RQ_L(true, true); else BBC_RQ_L(true, false); }
  else { if (na) BBC_RQ_L(false, true); else BBC_RQ_L(false, false); }
#undef BBC_RQ_L
}

// One PQ scan pass: work items (k_scan_plan), then one persistent CTA per SM over them.
// na: code loads bypass L1 allocation (codes larger than half of L2, or forced by
// bbc_set_code_loads).
void rq_scan(int M, bool est, int num_sms, cudaStream_t st, const Batch& b, const Dev& dv,
             const uint8_t* ct, const long long* tb, float* out, long long stride, int mode, bool na,
             bool sweep) {
  if (b.nq <= 0) return;
  if (sweep) {                                       // the visiting order of the main pass
    k_sweep_order<<<b.nq, kSelNT, 0, st>>>(b, dv);
    g_launches += 1;
  }
  k_scan_plan<<<1, 1024, 0, st>>>(b, mode, b.items, b.nitems, kRqE);
  g_launches += 1;
  if (sweep) {
    const int gi = 4 * num_sms;
    cudaMemsetAsync(b.icnt, 0, (size_t)(dv.nlist + 1) * 4, st);
    k_item_count<<<gi, 256, 0, st>>>(b, mode, kRqE, dv.nlist);
    k_item_offsets<<<1, 1024, 0, st>>>(b.icnt, dv.nlist);
    k_item_scatter<<<gi, 256, 0, st>>>(b);
    g_launches += 3;
  }
  switch (M) {
    case 8: launch_rq<8>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
    case 16: launch_rq<16>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
    case 24: launch_rq<24>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
    case 32: launch_rq<32>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
    case 48: launch_rq<48>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
    case 64: launch_rq<64>(est, num_sms, st, b, dv, ct, tb, out, stride, mode, na, sweep); break;
  }
}

template <int M>
void launch_q4(bool est, int grid, cudaStream_t st, const Batch& b, const Dev& dv, const uint8_t* ct,
               const long long* tb, float* out, long long stride, int mode) {
  if (est) k_pq4_scan<M, true><<<grid, kQ4NT, 0, st>>>(b, dv, ct, tb, out, stride, mode, b.items, b.nitems);
  else k_pq4_scan<M, false><<<grid, kQ4NT, 0, st>>>(b, dv, ct, tb, out, stride, mode, b.items, b.nitems);
}

// One 4-bit PQ scan pass: the same work items, two CTAs of 512 threads per SM.
void q4_scan(int M, bool est, int num_sms, cudaStream_t st, const Batch& b, const Dev& dv,
             const uint8_t* ct, const long long* tb, float* out, long long stride, int mode) {
  if (b.nq <= 0) return;
  k_scan_plan<<<1, 1024, 0, st>>>(b, mode, b.items, b.nitems, kQ4Item);
  g_launches += 1;
  const int grid = 2 * num_sms;
  switch (M) {
    case 8: launch_q4<8>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
    case 16: launch_q4<16>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
    case 24: launch_q4<24>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
    case 32: launch_q4<32>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
    case 48: launch_q4<48>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
    case 64: launch_q4<64>(est, grid, st, b, dv, ct, tb, out, stride, mode); break;
  }
}

// PQ scan pass of either code width
void pq_scan(const bbc_index_s* ix, bool est, cudaStream_t st, const Batch& b, const Dev& dv, float* out,
             long long stride, int mode) {
  if (ix->nbits == 4) {
    q4_scan(ix->M, est, ix->num_sms, st, b, dv, ix->codes_t, ix->tbase, out, stride, mode);
    return;
  }
  // codes that do not fit in L2 are streamed past L1 (see k_pq_scan_rq); L2 size queried at load
  const bool big = (double)ix->n_local * ix->M > 0.5 * (double)ix->l2_bytes;
  const bool na = ix->code_loads == BBC_CODES_STREAM || (ix->code_loads == BBC_CODES_AUTO && big);
  // sweep order (k_sweep_order) of the main pass for codes that do not fit in L2; the sample
  // pass (the nearest lists, shared by the queries of a locality region) keeps probe order
  const bool sweep = mode == 1 && (ix->scan_order == BBC_ORDER_SWEEP || (ix->scan_order == BBC_ORDER_AUTO && big));
  rq_scan(ix->M, est, ix->num_sms, st, b, dv, ix->codes_t, ix->tbase, out, stride, mode, na, sweep);
}

bbc_status check_args(bbc_index ix, const void* q, int64_t nq, int32_t k, int32_t nprobe,
                      int64_t budget, const void* oi, const void* od, const void* ws) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (ix->broken) return fail(BBC_ERR_STATE, "index handle unusable after an earlier CUDA error");
  if (nq < 0) return fail(BBC_ERR_ARG, "nq < 0");
  if (k < 1 || k > ix->N) return fail(BBC_ERR_ARG, "k must satisfy 1 <= k <= N");
  if (nprobe < 1 || nprobe > ix->nlist) return fail(BBC_ERR_ARG, "nprobe must satisfy 1 <= nprobe <= nlist");
  if (nprobe > kMaxProbe) return fail(BBC_ERR_ARG, "nprobe > 2048 is not supported");
  if (budget < k) return fail(BBC_ERR_ARG, "budget must be >= k");
  if (nq > 0 && (!q || !oi || !od || !ws)) return fail(BBC_ERR_ARG, "null pointer");
  return BBC_OK;
}

// ---------------------------------------------------------------------------------------------
// Collectives.  A search runs over one or more local shards; exchange steps call Comm.
//   GroupComm: G shards of one process on one device (element-wise reduction kernel)
//   NcclComm : one shard per process, ncclAllReduce on the search stream (NVLink/NVSwitch)
// ---------------------------------------------------------------------------------------------
enum class Dt { I32, U32, I64, F32 };
enum class Op { Sum, Min };

struct Comm {
  virtual ~Comm() {}
  virtual int world() const = 0;
  virtual bool allreduce(const std::vector<void*>& bufs, size_t n, Dt dt, Op op, cudaStream_t st) = 0;
  // host value -> its minimum over the processes of the communicator (synchronises `st`); the
  // shards of one process already agree
  virtual bool agree_min(long long* v, cudaStream_t st) { (void)v; (void)st; return true; }
  // all-gather with per-rank sizes of 8-byte elements: rank r's send[r] (count[r] elements) lands
  // at recv + displ[r] of the receiving rank(s) (for a single-process group: shard 0)
  virtual bool allgatherv(const std::vector<const void*>& send, const std::vector<void*>& recv,
                          const long long* count, const long long* displ, cudaStream_t st) = 0;
};

struct GroupComm : Comm {
  int G;
  explicit GroupComm(int g) : G(g) {}
  int world() const override { return G; }
  bool allreduce(const std::vector<void*>& bufs, size_t n, Dt dt, Op op, cudaStream_t st) override {
    if (n == 0) return true;
    GroupPtrs gp;
    for (int g = 0; g < G; ++g) gp.p[g] = bufs[g];
    const int blocks = (int)std::min<size_t>(4096, (n + 255) / 256);
    const int o = op == Op::Sum ? 0 : 1;
    switch (dt) {
      case Dt::I32: k_group_allreduce<int><<<blocks, 256, 0, st>>>(gp, G, (long long)n, o); break;
      case Dt::U32: k_group_allreduce<unsigned><<<blocks, 256, 0, st>>>(gp, G, (long long)n, o); break;
      case Dt::I64: k_group_allreduce<long long><<<blocks, 256, 0, st>>>(gp, G, (long long)n, o); break;
      case Dt::F32: k_group_allreduce<float><<<blocks, 256, 0, st>>>(gp, G, (long long)n, o); break;
    }
    g_launches += 1;
    return cudaGetLastError() == cudaSuccess;
  }
  bool allgatherv(const std::vector<const void*>& send, const std::vector<void*>& recv,
                  const long long* count, const long long* displ, cudaStream_t st) override {
    for (int r = 0; r < G; ++r)
      if (count[r] > 0 && cudaMemcpyAsync((unsigned long long*)recv[0] + displ[r], send[r], (size_t)count[r] * 8,
                                          cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return false;
    return true;
  }
};

struct NcclComm : Comm {
  ncclComm_t c;
  ncclComm_t cx;                      // second communicator: the result all-gather (copy stream)
  int W, me;
  long long* scratch;                 // one device int64 (bbc_comm_init)
  NcclComm(ncclComm_t comm, ncclComm_t commx, int w, int rank, long long* sc)
      : c(comm), cx(commx), W(w), me(rank), scratch(sc) {}
  int world() const override { return W; }
  bool allreduce(const std::vector<void*>& bufs, size_t n, Dt dt, Op op, cudaStream_t st) override {
    if (n == 0) return true;
    ncclDataType_t t = dt == Dt::I32 ? ncclInt32 : dt == Dt::U32 ? ncclUint32 : dt == Dt::I64 ? ncclInt64 : ncclFloat32;
    return ncclAllReduce(bufs[0], bufs[0], n, t, op == Op::Sum ? ncclSum : ncclMin, c, st) == ncclSuccess;
  }
  bool agree_min(long long* v, cudaStream_t st) override {
    if (W == 1) return true;
    return cudaMemcpyAsync(scratch, v, 8, cudaMemcpyHostToDevice, st) == cudaSuccess &&
           ncclAllReduce(scratch, scratch, 1, ncclInt64, ncclMin, c, st) == ncclSuccess &&
           cudaMemcpyAsync(v, scratch, 8, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
           cudaStreamSynchronize(st) == cudaSuccess;
  }
  // grouped broadcasts, one per root rank: an all-gather with per-rank sizes
  bool allgatherv(const std::vector<const void*>& send, const std::vector<void*>& recv,
                  const long long* count, const long long* displ, cudaStream_t st) override {
    if (ncclGroupStart() != ncclSuccess) return false;
    bool ok = true;
    for (int r = 0; r < W && ok; ++r) {
      if (count[r] == 0) continue;
      unsigned long long* dst = (unsigned long long*)recv[0] + displ[r];
      ok = ncclBroadcast(r == me ? send[0] : (const void*)dst, dst, (size_t)count[r], ncclUint64, r, cx, st) ==
           ncclSuccess;
    }
    return ncclGroupEnd() == ncclSuccess && ok;
  }
};

struct Shard {
  RbqBufs rb;
  XBuf xb;
  bbc_index_s* ix;
  char* ws;
  size_t ws_bytes;
  Plan p;
  Dev dv;
  Batch b;
  DistBuf db;
  float* qstage;
  long long* oids;
  float* od2;
  int rank;
};

// ------------------------------------------------------------------ stage launchers (one shard)
void stage_probe(Shard& s, cudaStream_t st) {
  bbc_index_s* ix = s.ix;
  StageScope sc(ix, st, BBC_STAGE_PROBE);
  if (s.dv.probe_tc && ix->probe_ws_ok) {
    const int qt = (s.b.nq + kTcM - 1) / kTcM;
    const int stripes = std::max(1, std::min((ix->nlist + kTcN - 1) / kTcN, ix->num_sms / std::max(1, qt)));
    set_smem(k_probe_mma_ws, kPwSmem);
    if (qt > 0)
      k_probe_mma_ws<<<qt * stripes, kPwNT, kPwSmem, st>>>(s.b.Q, ix->cmu, ix->cnorm, s.b.coarse, s.b.nq,
                                                         ix->nlist, ix->d, stripes, ix->ptm_hi, ix->ptm_lo);
  } else if (s.dv.probe_tc) {
    const dim3 gt((ix->nlist + kTcN - 1) / kTcN, (s.b.nq + kTcM - 1) / kTcM);
    set_smem(k_probe_mma, kTcSmem);
    k_probe_mma<<<gt, kTcNT, kTcSmem, st>>>(s.b.Q, ix->centroids, ix->cmu, ix->cnorm, s.b.coarse,
                                            s.b.nq, ix->nlist, ix->d);
  } else {
    dim3 g1((ix->nlist + kPT - 1) / kPT, (s.b.nq + kPT - 1) / kPT);
    if (ix->metric == BBC_METRIC_IP)
      k_probe_d2<true><<<g1, 256, 0, st>>>(s.b.Q, ix->centroids, s.b.coarse, s.b.nq, ix->nlist, ix->d);
    else
      k_probe_d2<false><<<g1, 256, 0, st>>>(s.b.Q, ix->centroids, s.b.coarse, s.b.nq, ix->nlist, ix->d);
  }
  k_probe_select<<<s.b.nq, kSelNT, 0, st>>>(s.b, s.dv);
  g_launches += 2;
  if (s.b.nq > 0) {
    int P2 = 1;
    while (P2 < s.b.nq) P2 <<= 1;
    if (P2 <= kQpermMax) {
      set_smem(k_qperm, (size_t)P2 * 8);
      k_qperm<<<1, 1024, (size_t)P2 * 8, st>>>(s.b, ix->lrank, const_cast<int*>(s.b.qperm));
    } else {
      k_iota<<<(s.b.nq + 255) / 256, 256, 0, st>>>(const_cast<int*>(s.b.qperm), s.b.nq);
    }
    g_launches += 1;
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda): a 2-D map
// [rows x cols] of esize-byte elements (row stride = cols elements) with boxes of box_rows x
// box_cols and 128-byte swizzle.
bool encode_tmap(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t cols,
                 uint64_t rows, uint32_t box_cols, uint32_t box_rows) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<Fn>(f);
  }
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {cols * esize};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// RaBitQ tensor-core path, after the probe: the pair layout (slots grouped by list, sample pairs
// first, each list's slot range padded to a multiple of kRbN) and every estimated pair's query
// code + record at its slot.
void rbq_pairs(Shard& s, const Batch& b, cudaStream_t st) {
  bbc_index_s* ix = s.ix;
  const long long pairs = (long long)b.nq * b.nprobe;
  if (pairs == 0) return;
  const unsigned gp = (unsigned)((pairs + 255) / 256);
  cudaMemsetAsync(s.rb.cnt_m, 0, (size_t)(ix->nlist + 1) * 4, st);
  cudaMemsetAsync(s.rb.cnt_s, 0, (size_t)(ix->nlist + 1) * 4, st);
  k_rbq_lcount<<<gp, 256, 0, st>>>(b, s.dv, s.rb.cnt_m, s.rb.cnt_s);
  k_rbq_lscan<<<1, 1024, 0, st>>>(s.rb.cnt_m, s.rb.cnt_s, s.rb.off, s.rb.cur_s, s.rb.cur_m, ix->nlist);
  k_rbq_lfill<<<gp, 256, 0, st>>>(b, s.dv, s.rb.cur_s, s.rb.cur_m, s.rb.islot);
  set_smem(k_rbq_pairs, (size_t)ix->D * 4);
  k_rbq_pairs<<<dim3((b.nprobe + kPairsPerCta - 1) / kPairsPerCta, b.nq), 256, (size_t)ix->D * 4, st>>>(
      b, s.dv, s.rb.islot, s.rb.qbar, s.rb.pinfo);
  g_launches += 4;
}

void stage_tables(Shard& s, cudaStream_t st) {
  bbc_index_s* ix = s.ix;
  StageScope sc(ix, st, BBC_STAGE_TABLES);
  if (ix->kind == BBC_KIND_PQ) {
    k_pq_lut<<<dim3(ix->M, s.b.nq), 1 << ix->nbits, 0, st>>>(s.b, s.dv);
    if (ix->nbits == 4) {
      k_pq4_qlut<<<s.b.nq, ix->M * 16, 0, st>>>(s.b, s.dv);
      g_launches += 1;
    }
  } else if ((size_t)ix->d * 4 * 8 <= 48 * 1024) {
    k_rbq_rotate<8><<<dim3((ix->D + kRotNT - 1) / kRotNT, (s.b.nq + 7) / 8), kRotNT, (size_t)ix->d * 4 * 8, st>>>(s.b, s.dv);
  } else {
    set_smem(k_rbq_rotate<1>, (size_t)ix->d * 4);
    k_rbq_rotate<1><<<dim3((ix->D + kRotNT - 1) / kRotNT, s.b.nq), kRotNT, (size_t)ix->d * 4, st>>>(s.b, s.dv);
  }
  g_launches += 1;
  if (ix->kind == BBC_KIND_RABITQ && ix->rbq_tc) rbq_pairs(s, s.b, st);
}

// RaBitQ tensor-core pass over the selected (query, list) pairs: inverted index + list-major GEMM
void rbq_tc_pass(Shard& s, const Batch& b, cudaStream_t st, bool sample) {
  bbc_index_s* ix = s.ix;
  const long long pairs = (long long)b.nq * b.nprobe;
  if (pairs == 0 || ix->rbq_ntiles == 0) return;
  if (!sample) {
    k_rbq_paircell<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(b, s.rb.islot, s.rb.pinfo);
    g_launches += 1;
  }
  RbqTc t{s.rb.qbar, s.rb.pinfo, s.rb.off, s.rb.cnt_s, s.rb.cnt_m, ix->rbq_tiles, ix->rbq_pc};
  // TMA map of the query codes: [slots x D] bytes, boxes of 32 rows x 128 B, 128-byte swizzle
  const long long slots = pairs + (long long)kRbN * ix->nlist;
  CUtensorMap tm;
  if (!encode_tmap(&tm, s.rb.qbar, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)ix->D, (uint64_t)slots, 128, kRbN)) {
    ix->broken = true;                               // reported by the CU check after the stage
    return;
  }
  // nst = 2 query-tile stages of kRbN pairs (A lives in tensor memory; shared memory holds the B
  // stages and the kRbRec-deep records ring)
  const int nkb = (ix->D + 127) / 128;
  auto ws_smem = [&](int nst) {
    return (size_t)nst * nkb * kRbN * 128 + (size_t)kRbRec * kRbN * sizeof(RbqPair) + 3 * kRbM * 4 +
           (size_t)(2 * nst + 2 * kRbRec + 4) * 8 + 16;
  };
  const int nst = 2;
  const size_t smw = ws_smem(nst);
  if (sample) {
    set_smem(k_rbq_mma_ws<true>, smw);
    k_rbq_mma_ws<true><<<ix->rbq_ntiles, kRbWsNT, smw, st>>>(b, s.dv, t, nst, tm);
  } else {
    set_smem(k_rbq_mma_ws<false>, smw);
    k_rbq_mma_ws<false><<<ix->rbq_ntiles, kRbWsNT, smw, st>>>(b, s.dv, t, nst, tm);
    // the histogram from the ids afterwards: formed in the GEMM epilogue with one global
    // reduction per counted object it was slower (C3 Push 2.10 -> 2.99 ms: the counted ids of a
    // query crowd a few cells)
    k_cell_hist<<<dim3(std::max(1, (8 * ix->num_sms + b.nq - 1) / b.nq), b.nq), 256, 0, st>>>(b);
    g_launches += 1;
  }
  g_launches += 1;
}


// a3: estimates of the (local) sample objects -> val
void stage_sample_est(Shard& s, cudaStream_t st) {
  bbc_index_s* ix = s.ix;
  StageScope sc(ix, st, BBC_STAGE_SAMPLE);
  if (ix->kind == BBC_KIND_PQ) {
    pq_scan(ix, true, st, s.b, s.dv, s.b.val, s.p.cap, 0);
  } else if (ix->rbq_tc) {
    rbq_tc_pass(s, s.b, st, true);
  } else {
    const size_t sm = (size_t)ix->D * 4 + 4 * (ix->D / 32) * 4;
    set_smem(k_rbq_scan<true>, sm);
    k_rbq_scan<true><<<dim3(std::min(s.b.nprobe, 4), s.b.nq), kScanNT, sm, st>>>(s.b, s.dv, 1);
  }
  g_launches += 1;
}

// a4: bucket ids + local histogram of every probed object (sample ids from stored estimates:
// here when the edges were all-reduced, else already by k_select_edges<true>)
void stage_scan(Shard& s, cudaStream_t st, bool sample_cells) {
  bbc_index_s* ix = s.ix;
  const int nb = s.b.nq, nprobe = s.b.nprobe;
  if (ix->kind == BBC_KIND_PQ && sample_cells) {  // the sample objects' ids: timed with the sample stage
    StageScope sc2(ix, st, BBC_STAGE_SAMPLE);
    k_sample_cells<<<dim3(8, nb), 256, 0, st>>>(s.b);
    g_launches += 1;
  }
  StageScope sc(ix, st, BBC_STAGE_SCAN);
  if (ix->kind == BBC_KIND_PQ) {
    pq_scan(ix, false, st, s.b, s.dv, nullptr, 0, 1);
    g_launches += 1;
    if (s.b.early) {
      // Algorithm 4 l.9-11: exact distances of the objects below tau_pred, as soon as the pass
      // has written the bucket ids and before Update/Collect (timed with the scan stage)
      const int nchunk = (int)((s.p.cap + kChunk - 1) / kChunk);
      k_early_rows<<<dim3(std::min(nchunk, 24), nb), kCmpNT, 0, st>>>(s.b, s.dv);
      g_launches += 1;
    }
  } else if (ix->rbq_tc) {
    rbq_tc_pass(s, s.b, st, false);
  } else {
    const int cta_per_q = std::max(1, std::min(nprobe, (3 * 148 * 6 + nb - 1) / nb));
    const int Gf = (nprobe + cta_per_q - 1) / cta_per_q;
    const size_t sm = (size_t)ix->D * 4 + 4 * (ix->D / 32) * 4;
    set_smem(k_rbq_scan<false>, sm);
    k_rbq_scan<false><<<dim3((nprobe + Gf - 1) / Gf, nb), kScanNT, sm, st>>>(s.b, s.dv, Gf);
    g_launches += 1;
  }
}

// AUTO: list order when each row is, on average, a candidate of >= 4 queries of the micro-batch
// (nq * budget / N): the queries of a list then share its rows through L2 (C2 0.93 -> 0.90 ms,
// C3 11.2 -> 6.6, C4 49.8 -> 25.3); query order otherwise (C5: ~3 queries per row, list order
// 11 % slower -- its segment and query-vector overheads are not repaid).
bool rerank_list_order(const bbc_index_s* ix, const Batch& b, int rowb) {
  (void)rowb;
  if (ix->rerank_order != BBC_RERANK_AUTO)
    return ix->rerank_order == BBC_RERANK_LIST || ix->rerank_order == BBC_RERANK_TILE;
  const double reuse = (double)b.nq * (double)b.budget / std::max<double>(1.0, (double)ix->n_local);
  return reuse >= 4.0;
}

// list order with the list's rows staged in shared memory tile by tile (bbc_rerank_tile.cuh):
// available for fp32 rows of 128-512 bytes, on request only -- measured slower than the L2-fed
// list order (C4 25.4 -> 37.0 ms, C2 0.90 -> 1.51 ms), so AUTO does not take it
bool rerank_tile(const bbc_index_s* ix, const Batch& b, int rowb) {
  if (!ix->rt_units || ix->early || !rerank_list_order(ix, b, rowb)) return false;
  return ix->rerank_order == BBC_RERANK_TILE;
}

void stage_compact(Shard& s, cudaStream_t st) {
  StageScope sc(s.ix, st, BBC_STAGE_COMPACT);
  const int nb = s.b.nq;
  const int nchunk = (int)((s.p.cap + kChunk - 1) / kChunk);
  if (s.b.remap_m > 0) {
    k_remap<<<nb, 256, 0, st>>>(s.b);
    g_launches += 1;
  }
  k_tau<<<nb, 32, 0, st>>>(s.b);
  k_count<<<dim3(std::min((nchunk + kCntPer - 1) / kCntPer, 8), nb), kCmpNT, 0, st>>>(s.b, s.b.chunk, nchunk);
  k_chunk_offsets<<<nb, 256, 0, st>>>(s.b, s.b.chunk, nchunk);

  Batch be = s.b;                                   // segment starts only for the list-order re-rank
  if (!rerank_list_order(s.ix, s.b, s.ix->raw_u8 ? s.ix->d : s.ix->d * 4)) be.sstart = nullptr;
  if (s.b.early) k_emit<true><<<dim3(std::min(nchunk, 24), nb), kCmpNT, 0, st>>>(be, s.dv, s.b.chunk, nchunk);
  else k_emit<false><<<dim3(std::min(nchunk, 24), nb), kCmpNT, 0, st>>>(be, s.dv, s.b.chunk, nchunk);
  g_launches += 4;
}

// rows per lane group and 16-byte chunks per lane by row size; one row per lane group in flight
// and high occupancy (4 CTAs/SM) beat deeper per-warp unrolling (tuned on C2: 1.55 ms with 2
// rows in flight at 2 CTAs/SM -> 0.92 ms)
#ifndef BBC_RR_MINB512
#define BBC_RR_MINB512 4                                  // CTAs/SM of the <= 512-byte-row re-rank
#endif
#ifndef BBC_RR_STEPS512
#define BBC_RR_STEPS512 1                                 // rows in flight per lane group (ditto)
#endif
#define BBC_RR_VARIANTS(X)                                      \
  if (rowb <= 128) {                                            \
    if (u8) X(true, 8, 1, 4, 4);                                \
    else X(false, 8, 1, 4, 4);                                  \
  } else if (rowb <= 512) {                                     \
    if (u8) X(true, 8, 4, BBC_RR_STEPS512, BBC_RR_MINB512);     \
    else X(false, 8, 4, BBC_RR_STEPS512, BBC_RR_MINB512);       \
  } else if (rowb <= 1024) {                                    \
    X(false, 8, 8, 1, 3);                                       \
  } else {                                                      \
    X(false, 32, 8, 1, 3);                                      \
  }

// f1: Algorithm 3 in place of steps a4..a7 (bbc_alg3.cuh): estimates of every probed object
// (the RaBitQ scan in EST mode over all probed lists), then one CTA per query for the bounds,
// the two buffers and the marginal-bucket loop.  Candidates leave with exact d^2 (B_exact) or
// +inf, ready for k_final_select.
void stage_rerank(Shard& s, cudaStream_t st);
void stage_alg3(Shard& s, cudaStream_t st) {
  const bbc_index_s* ix = s.ix;
  Batch b2 = s.b;
  b2.nsamp = s.b.a3nall;
  {
    StageScope sc(s.ix, st, BBC_STAGE_SCAN);
    k_fill_int<<<(s.b.nq + 255) / 256, 256, 0, st>>>(b2.nsamp, s.b.nq, s.b.nprobe);
    g_launches += 1;
    if (ix->rbq_tc) {
      rbq_pairs(s, b2, st);
      rbq_tc_pass(s, b2, st, true);
    } else {
      const size_t sm = (size_t)ix->D * 4 + 4 * (ix->D / 32) * 4;
      set_smem(k_rbq_scan<true>, sm);
      k_rbq_scan<true><<<dim3(std::min(s.b.nprobe, 64), s.b.nq), kScanNT, sm, st>>>(b2, s.dv, 1);
      g_launches += 1;
    }
  }
  if (ix->alg3 == BBC_ALG3_LIST) {
    // list mode: bounds, tau and the candidates' lower-bound buckets (k_alg3<.., 1>), the
    // candidates {a_lb <= tau} compacted in probe order and their exact d^2 computed by the
    // list-order re-rank (a list's rows shared through L2 by its queries), then the loop on
    // bucket counts over those distances (k_alg3_loop)
    {
      StageScope sc(s.ix, st, BBC_STAGE_COMPACT);
      k_alg3<false, 1><<<s.b.nq, kA3NT, 0, st>>>(s.b, s.dv, ix->alg3_eps0);
      g_launches += 1;
    }
    {
      StageScope sc(s.ix, st, BBC_STAGE_COMPACT);
      const int nb = s.b.nq;
      const int nchunk = (int)((s.p.cap + kChunk - 1) / kChunk);
      k_count<<<dim3(std::min((nchunk + kCntPer - 1) / kCntPer, 8), nb), kCmpNT, 0, st>>>(s.b, s.b.chunk, nchunk);
      k_chunk_offsets<<<nb, 256, 0, st>>>(s.b, s.b.chunk, nchunk);
      Batch be = s.b;
      if (!rerank_list_order(s.ix, s.b, s.ix->raw_u8 ? s.ix->d : s.ix->d * 4)) be.sstart = nullptr;
      k_emit<false><<<dim3(std::min(nchunk, 24), nb), kCmpNT, 0, st>>>(be, s.dv, s.b.chunk, nchunk);
      g_launches += 3;
    }
    stage_rerank(s, st);
    StageScope sc(s.ix, st, BBC_STAGE_RERANK);
    k_alg3_loop<<<s.b.nq, kA3NT, 0, st>>>(s.b, s.dv);
    g_launches += 1;
    return;
  }
  StageScope sc(s.ix, st, BBC_STAGE_RERANK);
  const size_t sm = (size_t)ix->d * 4;
  if (ix->raw_u8) {
    set_smem(k_alg3<true, 0>, sm);
    k_alg3<true, 0><<<s.b.nq, kA3NT, sm, st>>>(s.b, s.dv, ix->alg3_eps0);
  } else {
    set_smem(k_alg3<false, 0>, sm);
    k_alg3<false, 0><<<s.b.nq, kA3NT, sm, st>>>(s.b, s.dv, ix->alg3_eps0);
  }
  g_launches += 1;
}

template <bool IP, bool ER = false>
void launch_rerank(Shard& s, dim3 g, cudaStream_t st, int rowb) {
  const bool u8 = s.ix->raw_u8 != 0;
#define BBC_RR_Q(U8, LPC, MAXV, STEPS, MINB) k_rerank<U8, LPC, MAXV, STEPS, MINB, IP, ER><<<g, kRrNT, 0, st>>>(s.b, s.dv)
  BBC_RR_VARIANTS(BBC_RR_Q)
#undef BBC_RR_Q
}

// Grid: about one warp per kRrSPW pieces.  Pieces <= segments + candidates / piece, segments
// <= nq * nprobe; candidates are taken as 1.5x the budget (|S*| is the budget plus part of the
// threshold bucket); the kernel strides by the grid, so an underestimate costs time, not results.
template <bool IP, int SPW, bool ER = false>
void launch_rerank_seg(Shard& s, cudaStream_t st, int rowb) {
  const bool u8 = s.ix->raw_u8 != 0;
  const long long nq = s.b.nq;
  const long long cand = std::min<long long>(s.p.cap, s.b.budget + s.b.budget / 2);
  const long long pieces = nq * s.b.nprobe + nq * cand / rr_piece(rowb);
  const long long per_cta = (kRrNT / 32) * SPW;
  const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((pieces + per_cta - 1) / per_cta,
                                                                           (1LL << 30) / per_cta));
  const int covered = (int)(grid * per_cta);
  const int* nseg = s.b.rs_off + s.ix->nlist;
#define BBC_RR_S(U8, LPC, MAXV, STEPS, MINB)                                                           \
  do {                                                                                                \
    k_rerank_seg<U8, LPC, MAXV, STEPS, MINB, IP, SPW, false, ER><<<grid, kRrNT, 0, st>>>(s.b, s.dv, s.b.rseg, nseg, 0); \
    k_rerank_seg<U8, LPC, MAXV, STEPS, MINB, IP, SPW, true, ER><<<2 * s.ix->num_sms, kRrNT, 0, st>>>(      \
        s.b, s.dv, s.b.rseg, nseg, covered);                                                          \
  } while (0)
  BBC_RR_VARIANTS(BBC_RR_S)
#undef BBC_RR_S
}

// segments per warp: 8 for rows >= 1 KB, else 4 (tuned: C3 3840 B rows 8 ~ 16 > 4 > 2 > 1; C4 384 B
// rows 4 > 8 > 2)
template <bool IP, bool ER = false>
void launch_rerank_list(Shard& s, cudaStream_t st, int rowb) {
  if (rowb >= 1024) launch_rerank_seg<IP, 8, ER>(s, st, rowb);
  else launch_rerank_seg<IP, 4, ER>(s, st, rowb);
}


void stage_rerank(Shard& s, cudaStream_t st) {
  bbc_index_s* ix = s.ix;
  StageScope sc(ix, st, BBC_STAGE_RERANK);
  const int nb = s.b.nq;
  const int rowb = ix->raw_u8 ? ix->d : ix->d * 4;
  const bool ip = ix->metric == BBC_METRIC_IP;
  if (rerank_list_order(ix, s.b, rowb)) {
    ix->rr_list_batches++;
    // segments (query, first candidate, length) counted, offset and placed by list
    const unsigned gp = (unsigned)(((long long)nb * s.b.nprobe + 255) / 256);
    if (rerank_tile(ix, s.b, rowb)) {
      // pieces per (list, tile) unit, then one CTA per unit over its staged rows
      const int nu = ix->rt_nunits;
      cudaMemsetAsync(s.b.rs_cnt, 0, (size_t)(nu + 1) * 4, st);
      k_rr_tile_pieces<false><<<gp, 256, 0, st>>>(s.b, s.dv, ix->rt_ubase, s.b.rs_cnt, s.b.rseg);
      k_inv_scan<<<1, 1024, 0, st>>>(s.b.rs_cnt, s.b.rs_off, s.b.rs_cur, nu);
      k_rr_tile_pieces<true><<<gp, 256, 0, st>>>(s.b, s.dv, ix->rt_ubase, s.b.rs_cur, s.b.rseg);
      const size_t smem = (size_t)rt_rows(rowb) * rowb;
#define BBC_RT(RB, IPV)                                                                          \
  do {                                                                                          \
    set_smem(k_rerank_tile<RB, IPV>, smem);                                                     \
    k_rerank_tile<RB, IPV><<<nu, kRtNT, smem, st>>>(s.b, s.dv, s.b.rseg, ix->rt_units, s.b.rs_off); \
  } while (0)
      if (rowb == 128) { if (ip) BBC_RT(128, true); else BBC_RT(128, false); }
      else if (rowb == 256) { if (ip) BBC_RT(256, true); else BBC_RT(256, false); }
      else if (rowb == 384) { if (ip) BBC_RT(384, true); else BBC_RT(384, false); }
      else { if (ip) BBC_RT(512, true); else BBC_RT(512, false); }
#undef BBC_RT
      g_launches += 4;
      return;
    }
    cudaMemsetAsync(s.b.rs_cnt, 0, (size_t)(ix->nlist + 1) * 4, st);
    k_rr_segments<false><<<gp, 256, 0, st>>>(s.b, s.b.rs_cnt, s.b.rseg, rr_piece(rowb));
    k_inv_scan<<<1, 1024, 0, st>>>(s.b.rs_cnt, s.b.rs_off, s.b.rs_cur, ix->nlist);
    k_rr_segments<true><<<gp, 256, 0, st>>>(s.b, s.b.rs_cur, s.b.rseg, rr_piece(rowb));
    if (s.b.early) {                                 // Algorithm 4: "re-rank remaining candidates"
      if (ip) launch_rerank_list<true, true>(s, st, rowb);
      else launch_rerank_list<false, true>(s, st, rowb);
    } else if (ip) launch_rerank_list<true>(s, st, rowb);
    else launch_rerank_list<false>(s, st, rowb);
    g_launches += 5;
    return;
  }
  // ~32 CTAs per SM in total: short CTAs keep every SM busy to the end (tuned on C2)
  const int gy = std::max(1, (32 * ix->num_sms + nb - 1) / nb);
  const dim3 g(gy, nb);
  if (s.b.early) {
    if (ip) launch_rerank<true, true>(s, g, st, rowb);
    else launch_rerank<false, true>(s, g, st, rowb);
  } else if (ip) launch_rerank<true>(s, g, st, rowb);
  else launch_rerank<false>(s, g, st, rowb);
  g_launches += 1;
}

// ------------------------------------------------------------------ sharded exchange steps
bool all_reduce(Comm* comm, std::vector<Shard>& sh, void* Shard::*unused, size_t n, Dt dt, Op op,
                cudaStream_t st, const std::function<void*(Shard&)>& ptr) {
  std::vector<void*> bufs;
  for (auto& s : sh) bufs.push_back(ptr(s));
  return comm->allreduce(bufs, n, dt, op, st);
}

bbc_status dist_edges(std::vector<Shard>& sh, Comm* comm, cudaStream_t st) {
  bbc_index_s* ix = sh[0].ix;
  const int nb = sh[0].b.nq;
  StageScope sc(ix, st, BBC_STAGE_COMM);
  for (auto& s : sh) {
    k_ds_edges_init<<<(nb + 255) / 256, 256, 0, st>>>(s.b, s.db);
    k_ds_localmin<<<nb, 256, 0, st>>>(s.b, s.db);
    g_launches += 2;
  }
  if (!all_reduce(comm, sh, nullptr, (size_t)nb, Dt::U32, Op::Min, st, [](Shard& s) { return (void*)s.db.umin; }))
    return fail(BBC_ERR_NCCL, "all-reduce (sample minimum) failed");
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (auto& s : sh) {
      CU_NOIX(cudaMemsetAsync(s.db.dh, 0, (size_t)nb * kCells * 4, st));
      k_ds_hist<false><<<dim3(8, nb), 256, 0, st>>>(s.b, s.db, shift);
      g_launches += 1;
    }
    if (!all_reduce(comm, sh, nullptr, (size_t)nb * kCells, Dt::I32, Op::Sum, st, [](Shard& s) { return (void*)s.db.dh; }))
      return fail(BBC_ERR_NCCL, "all-reduce (sample histogram) failed");
    for (auto& s : sh) {
      k_ds_pick<<<nb, 32, 0, st>>>(s.b, s.db, shift);
      g_launches += 1;
    }
  }
  for (auto& s : sh) {
    k_ds_edges_finish<<<(nb + 255) / 256, 256, 0, st>>>(s.b, s.db);
    g_launches += 1;
  }
  return BBC_OK;
}

bbc_status dist_hist(std::vector<Shard>& sh, Comm* comm, cudaStream_t st) {
  StageScope sc(sh[0].ix, st, BBC_STAGE_COMM);
  if (!all_reduce(comm, sh, nullptr, (size_t)sh[0].b.nq * kCells, Dt::I32, Op::Sum, st, [](Shard& s) { return (void*)s.b.hist; }))
    return fail(BBC_ERR_NCCL, "all-reduce (bucket histogram) failed");
  return BBC_OK;
}

// select, part 1 (search stream): global |S*| per query, the (d^2, id) threshold of the k
// smallest by 8 radix passes, the per-(rank, query) counts of selected pairs and their packed
// offsets (every rank computes every rank's offsets from the all-reduced counts).
bbc_status dist_select(std::vector<Shard>& sh, Comm* comm, cudaStream_t st) {
  bbc_index_s* ix = sh[0].ix;
  const int nb = sh[0].b.nq, W = comm->world();
  StageScope sc(ix, st, BBC_STAGE_SELECT);
  for (auto& s : sh) {
    k_ds_ncand<<<(nb + 255) / 256, 256, 0, st>>>(s.b, s.db);
    g_launches += 1;
  }
  if (!all_reduce(comm, sh, nullptr, (size_t)nb, Dt::I32, Op::Sum, st, [](Shard& s) { return (void*)s.db.tot; }))
    return fail(BBC_ERR_NCCL, "all-reduce (candidate count) failed");
  for (auto& s : sh) {
    k_ds_final_init<<<(nb + 255) / 256, 256, 0, st>>>(s.b, s.db);
    g_launches += 1;
  }
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (auto& s : sh) {
      CU_NOIX(cudaMemsetAsync(s.db.dh, 0, (size_t)nb * kCells * 4, st));
      k_ds_hist<true><<<dim3(8, nb), 256, 0, st>>>(s.b, s.db, shift);
      g_launches += 1;
    }
    if (!all_reduce(comm, sh, nullptr, (size_t)nb * kCells, Dt::I32, Op::Sum, st, [](Shard& s) { return (void*)s.db.dh; }))
      return fail(BBC_ERR_NCCL, "all-reduce (selection histogram) failed");
    for (auto& s : sh) {
      k_ds_pick<<<nb, 32, 0, st>>>(s.b, s.db, shift);
      g_launches += 1;
    }
  }
  for (auto& s : sh) {
    CU_NOIX(cudaMemsetAsync(s.db.cnt, 0, (size_t)W * nb * 4, st));
    k_ds_select<false><<<nb, kSelNT, 0, st>>>(s.b, s.db, s.rank, s.xb);
    g_launches += 1;
  }
  if (!all_reduce(comm, sh, nullptr, (size_t)W * nb, Dt::I32, Op::Sum, st, [](Shard& s) { return (void*)s.db.cnt; }))
    return fail(BBC_ERR_NCCL, "all-reduce (selected counts) failed");
  return BBC_OK;
}

// select, part 2 (search stream, after the previous micro-batch's exchange released the
// buffers): counts and packed offsets into the exchange buffer, this rank's pairs packed, the
// per-rank totals copied to pinned host memory (the exchange sizes); ev_x[0] marks them ready.
bbc_status dist_pack(std::vector<Shard>& sh, Comm* comm, cudaStream_t st) {
  bbc_index_s* ix = sh[0].ix;
  const int nb = sh[0].b.nq, W = comm->world();
  StageScope sc(ix, st, BBC_STAGE_SELECT);
  for (auto& s : sh) {
    k_ds_counts_scan<<<W, 1024, 0, st>>>(s.b, s.db, s.xb);
    k_ds_select<true><<<nb, kSelNT, 0, st>>>(s.b, s.db, s.rank, s.xb);
    g_launches += 2;
  }
  CU(cudaMemcpyAsync(ix->h_tot, sh[0].xb.tot, (size_t)W * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaEventRecord(ix->ev_done[0], st));
  return BBC_OK;
}

// A micro-batch whose pairs are packed, waiting for its all-gather (enqueued once the search
// stream has the next micro-batch's work queued, so the host wait does not idle the GPU).
struct PendingX {
  bool on = false;
  long long q0 = 0;
  int nb = 0, bi = 0;
};

// The all-gather of a packed micro-batch and the unpack into the output, on the copy stream
// (the second communicator); ev_copied[0] marks the exchange buffers free again.
bbc_status dist_exchange(std::vector<Shard>& sh, Comm* comm, const PendingX& px, int k, bool host,
                         int64_t* out_ids, float* out_d2) {
  bbc_index_s* ix = sh[0].ix;
  const int W = comm->world();
  cudaStream_t cs = ix->copy_stream;
  CU(cudaEventSynchronize(ix->ev_done[0]));            // the sizes (h_tot) are on the host
  Displs dp{};
  long long cnt[8], dsp[8], acc = 0;
  for (int r = 0; r < W; ++r) {
    cnt[r] = ix->h_tot[r];
    dsp[r] = acc;
    dp.d[r] = acc;
    acc += cnt[r];
  }
  if (acc > (long long)px.nb * k) return fail(BBC_ERR_STATE, "exchange larger than its buffer");
  CU(cudaStreamWaitEvent(cs, ix->ev_done[0], 0));
  std::vector<const void*> sends;
  std::vector<void*> recvs;
  for (auto& s : sh) {
    sends.push_back(s.xb.send);
    recvs.push_back(s.xb.recv);
  }
  {
    StageScope sc(ix, cs, BBC_STAGE_COMM);
    if (!comm->allgatherv(sends, recvs, cnt, dsp, cs)) return fail(BBC_ERR_NCCL, "all-gather (results) failed");
  }
  Shard& s0 = sh[0];
  long long* oi = host ? (px.bi ? s0.b.ostage2_ids : s0.oids) : (long long*)out_ids + px.q0 * k;
  float* od = host ? (px.bi ? s0.b.ostage2_d2 : s0.od2) : out_d2 + px.q0 * k;
  k_ds_unpack<<<px.nb, 256, 0, cs>>>(px.nb, k, W, s0.xb, dp, oi, od);
  g_launches += 1;
  if (host) {
    CU(cudaMemcpyAsync(out_ids + px.q0 * k, oi, (size_t)px.nb * k * 8, cudaMemcpyDeviceToHost, cs));
    CU(cudaMemcpyAsync(out_d2 + px.q0 * k, od, (size_t)px.nb * k * 4, cudaMemcpyDeviceToHost, cs));
  }
  CU(cudaEventRecord(ix->ev_copied[0], cs));
  return BBC_OK;
}

// ------------------------------------------------------------------ one search over local shards
bbc_status run(std::vector<Shard>& sh, Comm* comm, const float* queries, int64_t nq, int32_t k,
               int32_t nprobe, int64_t budget, int64_t* out_ids, float* out_d2, void* stream,
               bool host, const bbc_debug_bufs* dbg) {
  for (auto& s : sh) {
    bbc_status st0 = check_args(s.ix, queries, nq, k, nprobe, budget, out_ids, out_d2, s.ws);
    if (st0 != BBC_OK) return st0;
  }
  if (comm != nullptr)
    for (auto& s : sh) {
      if (s.ix->alg3) return fail(BBC_ERR_ARG, "Algorithm 3 (bbc_set_bound_rerank) is single-shard only");
      if (s.ix->early) return fail(BBC_ERR_ARG, "Algorithm 4 (bbc_set_early_rerank) is single-shard only");
    }
  if (nq == 0) return BBC_OK;
  bbc_index_s* ix = sh[0].ix;                       // for CU() error marking
  CU(cudaSetDevice(ix->device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool dist = comm != nullptr;
  const int W = dist ? comm->world() : 1;
  long long nqb = nq;
  for (auto& s : sh) {
    s.p = make_plan(s.ix, nprobe, k, W, dist);
    if (s.ws_bytes < s.p.fixed + s.p.per_query)
      return fail(BBC_ERR_ARG, "workspace smaller than bbc_workspace_size min_bytes");
    nqb = std::min<long long>(nqb, (long long)((s.ws_bytes - s.p.fixed) / s.p.per_query));
  }
  // every rank must cut the batch into the same micro-batches (the collectives of each must
  // match): the per-query scratch depends on the local list sizes, so agree on the minimum
  if (dist && !comm->agree_min(&nqb, st)) return fail(BBC_ERR_NCCL, "all-reduce (micro-batch size) failed");
  if (dbg && nqb < nq) return fail(BBC_ERR_ARG, "debug search needs all queries in one micro-batch");
  // host path: the device->host copy of micro-batch i (copy stream) overlaps the search of
  // micro-batch i+1; outputs alternate between two staging buffers.  At least 4 micro-batches
  // (of >= 256 queries) so that most of the copy time is hidden.
  // The output copy against the work per query (code bytes of the nprobe largest lists plus the
  // budget's raw rows).  Where the copy is < 1/1000 of the work (C3: 60 KB vs ~230 MB) it is not
  // worth splitting the batch for (one micro-batch, copy exposed: C3 e2e 49k -> 65k -> 73k);
  // otherwise the tail halves down to nqb / 4 (C2: 150k -> 158k; measured divisors 1, 2, 4, 8).
  const double code_b = ix->kind == BBC_KIND_PQ ? (ix->nbits == 4 ? ix->M / 2.0 : (double)ix->M)
                                                : ix->D / 8.0 + 8.0;
  const double work_b = (double)sh[0].p.cap * code_b + (double)std::min<long long>(budget, ix->N) *
                                                           (ix->raw_u8 ? ix->d : 4.0 * ix->d);
  const int tail_div = (double)k * 12.0 * 1000.0 < work_b ? 1 : 4;
  const bool pipe = host && !dist && !dbg && tail_div > 1;
  // host-path micro-batches of nq/12 queries (at least 512): the copies of one overlap the search
  // of the next at a fine grain (C4: nq/2 -> nq/8: 140.7 -> 126.4 ms per 10,000 queries; with the
  // sweep-ordered scan nq/12 128.0 vs nq/8 131.6, nq/16 128.9, nq/6 135.0; C2's 1,000 queries
  // keep 512-query batches: smaller ones cost more than they overlap)
  if (pipe) nqb = std::min<long long>(nqb, std::max<long long>(512, (nq + 11) / 12));
  if ((pipe || dist) && !ix->copy_stream) {
    CU(cudaStreamCreateWithFlags(&ix->copy_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ix->copy_stream2, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) CU(cudaEventCreateWithFlags(&ix->ev_copied2[i], cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&ix->ev_done[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ix->ev_copied[i], cudaEventDisableTiming));
    }
  }
  if (dist && !ix->h_tot) CU(cudaHostAlloc((void**)&ix->h_tot, 8 * sizeof(long long), cudaHostAllocDefault));
  PendingX px;                                        // sharded: micro-batch awaiting its all-gather
  bool xbusy = false;                                 // an all-gather is enqueued on the copy stream
  int mb_index = 0;
  const long long budget_c = std::min<long long>(budget, (long long)1 << 40);
  for (auto& s : sh) {
    CU(cudaMemsetAsync(s.ix->stats, 0, kNStats * sizeof(long long), st));
    s.ix->microbatches = 0;
    s.ix->rr_list_batches = 0;
    if (s.ix->timing) s.ix->timed_calls++;
    s.dv = dev_view(s.ix);
    // a1 on the tensor cores when it wins: the shortlist re-score reads nprobe centroid rows per
    // query, the SIMT tiled kernel all nlist: tensor cores for nprobe <= nlist/16
    // (C4 at nlist/21: 4.15 -> 3.44 ms; at nlist/16 even; C2 at nlist/5.3 and C3 at nlist/2 SIMT)
    const int pm = s.ix->probe_mode;
    s.dv.probe_tc = s.ix->probe_tc_ok &&
                    (pm == BBC_PROBE_TENSOR || (pm == BBC_PROBE_AUTO && 16LL * nprobe <= s.ix->nlist));
  }
  // host path: the tail of the batch is cut into halving micro-batches so that the one
  // device->host copy left exposed, the last micro-batch's, is small.
  const long long min_nb = std::max<long long>(32, nqb / tail_div);
  int nb = 0;
  for (long long q0 = 0; q0 < nq; q0 += nb) {
    const long long rem = nq - q0;
    nb = (int)(pipe ? std::min<long long>(nqb, std::max<long long>(std::min(rem, min_nb), (rem + 1) / 2))
                    : std::min<long long>(nqb, rem));
    // host path: a ramped head too (nqb/4, then nqb/2), so that the first device->host copy starts
    // early -- when the copies are the longer stream (C4: 6 GB of results per step) the exposed
    // time is the first micro-batch's search plus the last one's copy
    if (pipe && mb_index < 2)
      nb = (int)std::min<long long>(nb, std::max<long long>(std::min(rem, min_nb), nqb >> (2 - mb_index)));
    for (auto& s : sh) {
      carve(s.ix, s.p, nb, (int)nqb, nprobe, s.ws, s.b, &s.qstage, &s.oids, &s.od2, k, &s.db, W, &s.rb,
            dist ? &s.xb : nullptr);
      Batch& b = s.b;
      b.nq = nb; b.nprobe = nprobe; b.k = k; b.budget = budget_c; b.cap = s.p.cap;
      b.nbuckets = s.ix->nbuckets;
      b.remap_m = s.ix->remap_m;
      b.stats = s.ix->stats;
      if (host) {
        CU(cudaMemcpyAsync(s.qstage, queries + q0 * ix->d, (size_t)nb * ix->d * 4,
                           cudaMemcpyHostToDevice, st));
        b.Q = s.qstage;
      } else {
        b.Q = queries + q0 * ix->d;
        if (!dist) {
          s.oids = (long long*)out_ids + q0 * k;
          s.od2 = out_d2 + q0 * k;
        }
      }
      CU(cudaMemsetAsync(b.hist, 0, (size_t)nb * kCells * 4, st));
      stage_probe(s, st);
      stage_tables(s, st);
      stage_sample_est(s, st);
      if (s.ix->broken) return fail(BBC_ERR_CUDA, "cuTensorMapEncodeTiled failed (RaBitQ query codes)");
    }
    if (!dist) {
      Shard& s = sh[0];
      {
        StageScope sc(s.ix, st, BBC_STAGE_SAMPLE);
        // the sample objects' bucket ids stay a separate wide kernel (k_sample_cells): fused
        // into this one-CTA-per-query select they cost more (C4: 2.5 + 1.5 -> 4.4 ms)
        set_smem(k_select_edges, kFsSmem);
        k_select_edges<<<nb, kSelNT, kFsSmem, st>>>(s.b, s.dv);
        g_launches += 1;
        if (s.b.early) {                              // Algorithm 4 l.4: the predicted threshold bucket
          set_smem(k_tau_pred, kFsSmem);
          k_tau_pred<<<nb, kSelNT, kFsSmem, st>>>(s.b, s.dv);
          g_launches += 1;
        }
      }
      if (s.ix->alg3) {
        stage_alg3(s, st);
      } else {
        stage_scan(s, st, true);
        stage_compact(s, st);
        stage_rerank(s, st);
      }
      const int bi = mb_index & 1;
      if (pipe) {
        if (bi == 1) { s.oids = s.b.ostage2_ids; s.od2 = s.b.ostage2_d2; }
        if (mb_index >= 2) CU(cudaStreamWaitEvent(st, ix->ev_copied[bi], 0));   // buffer free
      }
      {
        StageScope sc(s.ix, st, BBC_STAGE_SELECT);
        if (s.b.budget >= 50000) k_final_select<13><<<nb, kSelNT, 0, st>>>(s.b, s.dv, s.oids, s.od2);
        else k_final_select<11><<<nb, kSelNT, 0, st>>>(s.b, s.dv, s.oids, s.od2);
        g_launches += 1;
      }
      if (pipe) {
        // ids and distances on two copy streams (two copy engines in flight on the PCIe link)
        cudaStream_t cs = ix->copy_stream, cs2 = ix->copy_stream2;
        CU(cudaEventRecord(ix->ev_done[bi], st));
        CU(cudaStreamWaitEvent(cs, ix->ev_done[bi], 0));
        CU(cudaStreamWaitEvent(cs2, ix->ev_done[bi], 0));
        CU(cudaMemcpyAsync(out_ids + q0 * k, s.oids, (size_t)nb * k * 8, cudaMemcpyDeviceToHost, cs));
        CU(cudaMemcpyAsync(out_d2 + q0 * k, s.od2, (size_t)nb * k * 4, cudaMemcpyDeviceToHost, cs2));
        CU(cudaEventRecord(ix->ev_copied2[bi], cs2));
        CU(cudaStreamWaitEvent(cs, ix->ev_copied2[bi], 0));   // ev_copied: both copies done
        CU(cudaEventRecord(ix->ev_copied[bi], cs));
      }
    } else {
      bbc_status e = dist_edges(sh, comm, st);
      if (e != BBC_OK) return e;
      for (auto& s : sh) stage_scan(s, st, true);
      if ((e = dist_hist(sh, comm, st)) != BBC_OK) return e;
      for (auto& s : sh) {
        stage_compact(s, st);
        stage_rerank(s, st);
      }
      if ((e = dist_select(sh, comm, st)) != BBC_OK) return e;
      // the previous micro-batch's all-gather, now that this one's work is queued ahead of the
      // host wait; this micro-batch's packing waits until that exchange released the buffers
      if (px.on) {
        if ((e = dist_exchange(sh, comm, px, k, host, out_ids, out_d2)) != BBC_OK) return e;
        xbusy = true;
        px.on = false;
      }
      if (xbusy) CU(cudaStreamWaitEvent(st, ix->ev_copied[0], 0));
      if ((e = dist_pack(sh, comm, st)) != BBC_OK) return e;
      px.on = true;
      px.q0 = q0;
      px.nb = nb;
      px.bi = mb_index & 1;
    }
    CU(cudaGetLastError());
    Shard& s0 = sh[0];
    if (dbg) {
      const Batch& b = s0.b;
      auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
        return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st) : cudaSuccess;
      };
      CU(cp(dbg->probe, b.probe, (size_t)nb * nprobe * 4));
      CU(cp(dbg->rq2, b.rq2, (size_t)nb * nprobe * 4));
      CU(cp(dbg->nsample, b.nsamp, (size_t)nb * 4));
      CU(cp(dbg->edges, b.edges, (size_t)nb * 8));
      CU(cp(dbg->hist, b.hist, (size_t)nb * kCells * 4));
      CU(cp(dbg->tau, b.tau, (size_t)nb * 4));
      CU(cp(dbg->n_cand, b.ncand, (size_t)nb * 4));
      if (dbg->n_probed)
        CU(cudaMemcpy2DAsync(dbg->n_probed, 4, b.poff + nprobe, (size_t)(nprobe + 1) * 4, 4, nb,
                             cudaMemcpyDeviceToDevice, st));
      if (dbg->cand_ids || dbg->cand_d2) {
        k_debug_cands<<<dim3(64, nb), 256, 0, st>>>(b.cid, b.val, b.ncand, s0.p.cap,
                                                    (long long*)dbg->cand_ids, dbg->cand_d2, dbg->cand_stride,
                                                    b.early ? b.cpos : nullptr, dbg->cand_early);
        g_launches += 1;
      }
      if (dbg->tau_pred) {
        if (b.tpred) CU(cp(dbg->tau_pred, b.tpred, (size_t)nb * 4));
        else CU(cudaMemsetAsync(dbg->tau_pred, 0, (size_t)nb * 4, st));
      }
      if (dbg->est) {
        // every estimate in probe order, written to the caller's buffer (debug only)
        if (ix->kind == BBC_KIND_PQ) {
          pq_scan(ix, true, st, b, s0.dv, dbg->est, dbg->est_stride, 2);
        } else {
          Batch b2 = b;
          b2.val = dbg->est;
          b2.cap = dbg->est_stride;
          std::vector<int> all(nb, nprobe);
          int* ns_all = b.tau;  // scratch: tau was copied out above
          CU(cudaMemcpyAsync(ns_all, all.data(), (size_t)nb * 4, cudaMemcpyHostToDevice, st));
          CU(cudaStreamSynchronize(st));
          b2.nsamp = ns_all;
          if (ix->rbq_tc) {                           // pair records address b2's buffer
            rbq_pairs(s0, b2, st);
            rbq_tc_pass(s0, b2, st, true);
          } else {
            const size_t sm = (size_t)ix->D * 4 + 4 * (ix->D / 32) * 4;
            k_rbq_scan<true><<<dim3(std::min(nprobe, 64), nb), kScanNT, sm, st>>>(b2, s0.dv, 1);
          }
        }
        g_launches += 1;
        CU(cudaGetLastError());
      }
    }
    if (host && !pipe && !dist) {
      CU(cudaMemcpyAsync(out_ids + q0 * k, s0.oids, (size_t)nb * k * 8, cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(out_d2 + q0 * k, s0.od2, (size_t)nb * k * 4, cudaMemcpyDeviceToHost, st));
    }
    for (auto& s : sh) s.ix->microbatches++;
    ++mb_index;
  }
  if (px.on) {                                        // the last micro-batch's all-gather
    bbc_status e = dist_exchange(sh, comm, px, k, host, out_ids, out_d2);
    if (e != BBC_OK) return e;
    xbusy = true;
  }
  if (xbusy) CU(cudaStreamWaitEvent(st, ix->ev_copied[0], 0));   // results complete on `st`
  if (pipe)                                           // the caller's stream covers every copy
    for (int i = 0; i < std::min(mb_index, 2); ++i) CU(cudaStreamWaitEvent(st, ix->ev_copied[i], 0));
  if (host || dbg) CU(cudaStreamSynchronize(st));
  return BBC_OK;
}

bbc_status run_one(bbc_index ix, const float* queries, int64_t nq, int32_t k, int32_t nprobe,
                   int64_t budget, int64_t* out_ids, float* out_d2, void* workspace,
                   size_t ws_bytes, void* stream, bool host, const bbc_debug_bufs* dbg) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  std::vector<Shard> sh(1);
  sh[0].ix = ix;
  sh[0].ws = (char*)workspace;
  sh[0].ws_bytes = ws_bytes;
  sh[0].rank = ix->rank;
  if (ix->world > 1) {
    if (!ix->nccl) return fail(BBC_ERR_STATE, "sharded index: call bbc_comm_init first");
    NcclComm c((ncclComm_t)ix->nccl, (ncclComm_t)ix->nccl_x, ix->world, ix->rank, ix->nccl_scratch);
    return run(sh, &c, queries, nq, k, nprobe, budget, out_ids, out_d2, stream, host, dbg);
  }
  if (ix->force_dist) {                            // world-1 NCCL communicator (tests)
    if (!ix->nccl) return fail(BBC_ERR_STATE, "call bbc_comm_init first");
    NcclComm c((ncclComm_t)ix->nccl, (ncclComm_t)ix->nccl_x, 1, 0, ix->nccl_scratch);
    return run(sh, &c, queries, nq, k, nprobe, budget, out_ids, out_d2, stream, host, dbg);
  }
  return run(sh, nullptr, queries, nq, k, nprobe, budget, out_ids, out_d2, stream, host, dbg);
}

}  // namespace

template <int U>
__global__ void __launch_bounds__(256) k_l2_read(const uint4* __restrict__ buf, long long n16, int reps,
                                                 unsigned* __restrict__ sink) {
  unsigned acc = 0;
  const long long start = ((long long)blockIdx.x * 7919 * 256) % n16;
  for (int r = 0; r < reps; ++r) {
    for (long long i = threadIdx.x; i < n16; i += U * 256) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long k = start + i + u * 256;
        k = k >= n16 ? k - n16 : k;
        v[u] = i + u * 256 < n16 ? __ldcg(buf + k) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// ============================================================================================
// C ABI
// ============================================================================================
extern "C" {

const char* bbc_last_error(void) { return g_err.c_str(); }
int64_t bbc_launch_count(void) { return g_launches.load(); }

// L2 read roofline probe (k_l2_read: every CTA streams the whole L2-resident buffer with 16-byte
// loads, U in flight per thread, from a CTA-specific offset; after the first pass all reads hit L2).
bbc_status bbc_measure_l2_read(int32_t cuda_device, size_t bytes, int32_t reps, double* gbs) {
  if (!gbs || bytes < (1u << 20) || reps < 1) return fail(BBC_ERR_ARG, "bad arguments");
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(BBC_ERR_CUDA, "cudaSetDevice failed");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  void* buf = nullptr;
  unsigned* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) {
    cudaFree(buf);
    return fail(BBC_ERR_CUDA, "cudaMalloc failed");
  }
  cudaMemset(buf, 1, bytes);
  const long long n16 = (long long)(bytes / 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 4, 8 or 16 loads of 16 bytes in flight per thread and 4 or 8 CTAs of 256 threads per SM: the
  // best rate of the six (latency x bandwidth needs many bytes in flight per SM)
  double best = 0.0;
  cudaError_t err = cudaSuccess;
  for (int cfg = 0; cfg < 6 && err == cudaSuccess; ++cfg) {
    const int grid = sms * (cfg & 1 ? 8 : 4);
    auto launch = [&](int r) {
      if (cfg < 2) k_l2_read<4><<<grid, 256>>>((const uint4*)buf, n16, r, sink);
      else if (cfg < 4) k_l2_read<8><<<grid, 256>>>((const uint4*)buf, n16, r, sink);
      else k_l2_read<16><<<grid, 256>>>((const uint4*)buf, n16, r, sink);
    };
    launch(1);                                                          // warm L2
    cudaEventRecord(e0);
    launch(reps);
    cudaEventRecord(e1);
    err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 0.f) best = std::max(best, (double)grid * reps * (double)(n16 * 16) / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(sink);
  if (err != cudaSuccess || best <= 0.0) return fail(BBC_ERR_CUDA, "L2 probe failed");
  *gbs = best;
  return BBC_OK;
}

// Shared-memory lookup roofline probe: 32 warps per SM, each lane reading 4-byte words at
// conflict-free addresses (lane l -> bank l, as the replicated-LUT scan's lookups) with 32
// immediates off one base register per round, each read added into one of 8 fp32 sums: per
// lookup one LDS.32 (one wavefront per warp instruction) and one FADD, the scan's minimum.
__global__ void __launch_bounds__(1024, 1) k_lds_peak(int rounds, float* __restrict__ sink) {
  extern __shared__ __align__(16) float lsm[];                  // 128 KB
  for (int i = threadIdx.x; i < 32768; i += 1024) lsm[i] = (float)(i & 7);
  __syncthreads();
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(lsm) + 4u * (threadIdx.x & 31);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t off = 128u * (threadIdx.x >> 5);
#pragma unroll 1
  for (int r = 0; r < rounds; ++r) {
    const uint32_t a = s0 + off;
    static_for<32>([&](auto ic) {
      constexpr int u = decltype(ic)::value;
      float v;
      asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(u * 2048));
      acc[u & 7] += v;
    });
    off = (off + 128u * 33u) & 0xFFFFu;                         // a + 31 x 2048 + 124 < 128 KB
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += acc[i];
  if (t == -1.f) sink[0] = t;
}

bbc_status bbc_measure_smem_lookups(int32_t cuda_device, int32_t rounds, double* glookups) {
  if (!glookups || rounds < 1) return fail(BBC_ERR_ARG, "bad arguments");
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(BBC_ERR_CUDA, "cudaSetDevice failed");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return fail(BBC_ERR_CUDA, "cudaMalloc failed");
  const size_t smem = 128 << 10;
  cudaFuncSetAttribute(k_lds_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_lds_peak<<<sms, 1024, smem>>>(rounds / 10 + 1, sink);            // warm-up
  cudaEventRecord(e0);
  k_lds_peak<<<sms, 1024, smem>>>(rounds, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess || ms <= 0.f) return fail(BBC_ERR_CUDA, "shared-memory probe failed");
  *glookups = (double)sms * 1024.0 * 32.0 * (double)rounds / (ms * 1e-3) / 1e9;
  return BBC_OK;
}

bbc_status ivf_load(const char* path, int rank, int world, int cuda_device, bbc_index* out) {
  bbc_index_s* ix = nullptr;
  if (!path || !out) return fail(BBC_ERR_ARG, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(BBC_ERR_ARG, "bad rank/world");
  FILE* f = fopen(path, "rb");
  if (!f) return fail(BBC_ERR_IO, std::string("cannot open ") + path);
  char head[512];
  if (fread(head, 1, 512, f) != 512) { fclose(f); return fail(BBC_ERR_FORMAT, "short header"); }
  if (memcmp(head, "BBCIVF01", 8) != 0) { fclose(f); return fail(BBC_ERR_FORMAT, "bad magic"); }
  long long hdr[31], table[10][2];
  memcpy(hdr, head + 8, sizeof(hdr));
  memcpy(table, head + 256, sizeof(table));
  if (hdr[0] != 1) { fclose(f); return fail(BBC_ERR_FORMAT, "unsupported version"); }
  const int kind = (int)hdr[1], raw_u8 = (int)hdr[2];
  const long long N = hdr[3];
  const int d = (int)hdr[4], nlist = (int)hdr[5], M = (int)hdr[6], D = (int)hdr[8];
  if ((kind != BBC_KIND_PQ && kind != BBC_KIND_RABITQ) || N <= 0 || d <= 0 || nlist <= 0 ||
      N >= (1ll << 31)) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "bad header fields");
  }
  if (kind == BBC_KIND_PQ && (M <= 0 || d % M != 0 || M % 8 != 0 || M > 64 || (hdr[7] != 8 && hdr[7] != 4))) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "PQ needs 8- or 4-bit codes, M in {8,16,24,32,48,64}, M | d");
  }
  if (kind == BBC_KIND_RABITQ && (D % 64 != 0 || D < d)) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "RaBitQ needs D a multiple of 64, D >= d");
  }
  const int metric = (int)hdr[11];
  if (metric != BBC_METRIC_L2 && metric != BBC_METRIC_IP) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "unknown metric");
  }
  if (metric == BBC_METRIC_IP && kind != BBC_KIND_PQ) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "the inner-product metric is supported for PQ indexes only");
  }
  if (raw_u8 ? (d % 16 != 0 || d > 512) : (d % 4 != 0 || d > 1024)) {
    fclose(f);
    return fail(BBC_ERR_FORMAT, "d must be a multiple of 4 and <= 1024 (f32) or of 16 and <= 512 (u8)");
  }
  const size_t rowraw = (size_t)d * (raw_u8 ? 1 : 4);
  const size_t dsub = kind == BBC_KIND_PQ ? d / M : 0;
  const size_t expect[10] = {(size_t)nlist * d * 4, (size_t)(nlist + 1) * 8, (size_t)N * 8,
                             kind == BBC_KIND_PQ ? (size_t)M * ((size_t)1 << hdr[7]) * dsub * 4 : 0,
                             kind == BBC_KIND_PQ ? (size_t)N * M : 0,
                             kind == BBC_KIND_RABITQ ? (size_t)D * D * 4 : 0,
                             kind == BBC_KIND_RABITQ ? (size_t)nlist * D * 4 : 0,
                             kind == BBC_KIND_RABITQ ? (size_t)N * D / 8 : 0,
                             kind == BBC_KIND_RABITQ ? (size_t)N * 8 : 0, (size_t)N * rowraw};
  for (int s = 0; s < 10; ++s) {
    if (expect[s] && (size_t)table[s][1] != expect[s]) {
      fclose(f);
      return fail(BBC_ERR_FORMAT, "section " + std::to_string(s) + " has the wrong size");
    }
  }
  auto rd = [&](int s, void* dst, size_t off, size_t bytes) -> bool {
    if (fseeko(f, (off_t)(table[s][0] + off), SEEK_SET) != 0) return false;
    return fread(dst, 1, bytes, f) == bytes;
  };
  std::vector<long long> goff(nlist + 1);
  if (!rd(1, goff.data(), 0, goff.size() * 8)) { fclose(f); return fail(BBC_ERR_IO, "read offsets"); }
  if (goff[0] != 0 || goff[nlist] != N) { fclose(f); return fail(BBC_ERR_FORMAT, "bad list offsets"); }
  ix = new bbc_index_s();
  ix->device = cuda_device; ix->rank = rank; ix->world = world;
  ix->kind = kind; ix->d = d; ix->nlist = nlist; ix->M = M; ix->D = D; ix->raw_u8 = raw_u8;
  ix->nbits = kind == BBC_KIND_PQ ? (int)hdr[7] : 8;
  ix->metric = metric;
  ix->N = N;
  ix->gsize.resize(nlist);
  for (int L = 0; L < nlist; ++L) ix->gsize[L] = (int)(goff[L + 1] - goff[L]);
  // shard assignment: lists by (size desc, id asc), each to the least-loaded rank (ties: lowest)
  std::vector<int> owner(nlist, 0);
  if (world > 1) {
    std::vector<int> order(nlist);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return ix->gsize[a] > ix->gsize[b]; });
    std::vector<long long> load(world, 0);
    for (int L : order) {
      int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      owner[L] = r;
      load[r] += ix->gsize[L];
    }
  }
  ix->lsize.assign(nlist, 0);
  std::vector<long long> loff(nlist + 1, 0);
  for (int L = 0; L < nlist; ++L) {
    ix->lsize[L] = owner[L] == rank ? ix->gsize[L] : 0;
    loff[L + 1] = loff[L] + ix->lsize[L];
  }
  ix->n_local = loff[nlist];
  ix->max_list = *std::max_element(ix->gsize.begin(), ix->gsize.end());
  std::vector<int> sorted = ix->lsize;
  std::sort(sorted.begin(), sorted.end(), std::greater<int>());
  ix->desc_prefix.assign(nlist + 1, 0);
  for (int i = 0; i < nlist; ++i) ix->desc_prefix[i + 1] = ix->desc_prefix[i] + sorted[i];

  auto fail_load = [&](bbc_status s, const std::string& m) {
    fclose(f);
    ivf_free(ix);
    return fail(s, m);
  };
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail_load(BBC_ERR_CUDA, "cudaSetDevice");
  auto dalloc = [&](void** p, size_t bytes) -> bool {
    if (bytes == 0) bytes = 256;
    return cudaMalloc(p, bytes) == cudaSuccess;
  };
  // replicated arrays
  std::vector<char> buf;
  auto upload_full = [&](int s, void** dst) -> bool {
    size_t bytes = (size_t)table[s][1];
    buf.resize(bytes);
    if (!rd(s, buf.data(), 0, bytes)) return false;
    if (!dalloc(dst, bytes)) return false;
    return cudaMemcpy(*dst, buf.data(), bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  // per-object arrays: rows of owned lists, concatenated in list order
  auto upload_rows = [&](int s, size_t rowbytes, void** dst) -> bool {
    size_t bytes = (size_t)ix->n_local * rowbytes;
    if (!dalloc(dst, bytes)) return false;
    if (world == 1) {
      // stream in 256 MB chunks
      const size_t chunk = 256u << 20;
      buf.resize(std::min(bytes, chunk));
      for (size_t o = 0; o < bytes; o += chunk) {
        size_t nb = std::min(chunk, bytes - o);
        if (!rd(s, buf.data(), o, nb)) return false;
        if (cudaMemcpy((char*)*dst + o, buf.data(), nb, cudaMemcpyHostToDevice) != cudaSuccess) return false;
      }
      return true;
    }
    for (int L = 0; L < nlist; ++L) {
      if (!ix->lsize[L]) continue;
      size_t nb = (size_t)ix->lsize[L] * rowbytes;
      buf.resize(nb);
      if (!rd(s, buf.data(), (size_t)goff[L] * rowbytes, nb)) return false;
      if (cudaMemcpy((char*)*dst + (size_t)loff[L] * rowbytes, buf.data(), nb,
                     cudaMemcpyHostToDevice) != cudaSuccess)
        return false;
    }
    return true;
  };
  bool ok = upload_full(0, (void**)&ix->centroids);
  ok = ok && dalloc((void**)&ix->loff, (nlist + 1) * 8) &&
       cudaMemcpy(ix->loff, loff.data(), (nlist + 1) * 8, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && dalloc((void**)&ix->gsize_d, nlist * 4) &&
       cudaMemcpy(ix->gsize_d, ix->gsize.data(), nlist * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && upload_rows(2, 8, (void**)&ix->ids);
  if (kind == BBC_KIND_PQ) {
    ok = ok && upload_full(3, (void**)&ix->books);
    ok = ok && upload_rows(4, (size_t)M, (void**)&ix->codes);
  } else {
    ok = ok && upload_full(5, (void**)&ix->P);
    ok = ok && upload_full(6, (void**)&ix->wL);
    ok = ok && upload_rows(7, (size_t)D / 8, (void**)&ix->bits);
    ok = ok && upload_rows(8, 8, (void**)&ix->factors);
  }
  ok = ok && upload_rows(9, rowraw, &ix->raw);
  ok = ok && dalloc((void**)&ix->stats, kNStats * sizeof(long long));
  if (ok) {
    // centroid mean, |c - mu|^2 and max |c - mu| for the tensor-core probe's error bound
    std::vector<float> C((size_t)nlist * d);
    ok = cudaMemcpy(C.data(), ix->centroids, C.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    std::vector<double> mud(d, 0.0);
    for (int c = 0; c < nlist; ++c)
      for (int t = 0; t < d; ++t) mud[t] += C[(size_t)c * d + t];
    std::vector<float> mu(d), cn(nlist);
    for (int t = 0; t < d; ++t) mu[t] = (float)(mud[t] / nlist);
    double mx = 0.0;
    for (int c = 0; c < nlist; ++c) {
      double a = 0.0;
      for (int t = 0; t < d; ++t) {
        const double y = (double)(C[(size_t)c * d + t] - mu[t]);
        a += y * y;
      }
      cn[c] = (float)a;
      mx = std::max(mx, a);
    }
    ix->cmax = (float)(std::sqrt(mx) * (1.0 + 1e-6));
    // list regions for the query locality order: nearest of 256 evenly spaced pivot centroids
    const int npiv = std::min(256, nlist);
    std::vector<int> lr(nlist);
    for (int c = 0; c < nlist; ++c) {
      int best = 0;
      double bd = 1e300;
      for (int pv = 0; pv < npiv; ++pv) {
        const float* a = &C[(size_t)c * d];
        const float* bb = &C[(size_t)((long long)pv * nlist / npiv) * d];
        double s2 = 0.0;
        for (int t = 0; t < d; ++t) { const double y = (double)a[t] - bb[t]; s2 += y * y; }
        if (s2 < bd) { bd = s2; best = pv; }
      }
      lr[c] = (best << 20) | c;
    }
    ok = ok && dalloc((void**)&ix->lrank, (size_t)nlist * 4) &&
         cudaMemcpy(ix->lrank, lr.data(), (size_t)nlist * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && dalloc((void**)&ix->cmu, (size_t)d * 4) && dalloc((void**)&ix->cnorm, (size_t)nlist * 4) &&
         cudaMemcpy(ix->cmu, mu.data(), (size_t)d * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(ix->cnorm, cn.data(), (size_t)nlist * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    ix->probe_tc_ok = d <= kMaxDimTc && metric == BBC_METRIC_L2;
    if (ok && ix->probe_tc_ok && d <= 128 && d % 8 == 0) {
      // the TMA-fed probe (k_probe_mma_ws): centred centroids split hi/lo once, rows padded to 128
      const int npad = (nlist + kTcN - 1) / kTcN * kTcN;
      const size_t nb = (size_t)npad * d * 4;
      ok = dalloc((void**)&ix->pb_hi, nb) && dalloc((void**)&ix->pb_lo, nb);
      if (ok) {
        k_probe_split<<<(unsigned)(((long long)npad * d + 255) / 256), 256>>>(ix->centroids, ix->cmu, nlist,
                                                                              npad, d, ix->pb_hi, ix->pb_lo);
        ok = cudaDeviceSynchronize() == cudaSuccess;
      }
      ix->probe_ws_ok = ok && encode_tmap(&ix->ptm_hi, ix->pb_hi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)d,
                                          (uint64_t)npad, 32, kTcN) &&
                        encode_tmap(&ix->ptm_lo, ix->pb_lo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)d,
                                    (uint64_t)npad, 32, kTcN);
    }
  }
  if (ok && kind == BBC_KIND_RABITQ && D <= 1024 && D % 64 == 0) {
    std::vector<int2> tiles;
    for (int L = 0; L < nlist; ++L)
      for (int o = 0; o < ix->lsize[L]; o += kRbM) tiles.push_back(make_int2(L, o));
    ix->rbq_ntiles = (int)tiles.size();
    ok = dalloc((void**)&ix->rbq_pc, (size_t)std::max<long long>(1, ix->n_local) * 4) &&
         dalloc((void**)&ix->rbq_tiles, (size_t)std::max<size_t>(1, tiles.size()) * 8) &&
         cudaMemcpy(ix->rbq_tiles, tiles.data(), tiles.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && ix->n_local > 0) {
      k_rbq_popc<<<(unsigned)((ix->n_local + 255) / 256), 256>>>(ix->bits, ix->n_local, D, ix->rbq_pc);
      ok = cudaDeviceSynchronize() == cudaSuccess;
    }
    ix->rbq_tc = ok ? 1 : 0;
  }
  if (ok && !raw_u8 && (d * 4 == 128 || d * 4 == 256 || d * 4 == 384 || d * 4 == 512) && ix->n_local > 0) {
    // (list, tile) units of the shared-memory re-rank, in list order
    const int R = rt_rows(d * 4);
    std::vector<int2> units;
    std::vector<int> ubase(nlist);
    for (int L = 0; L < nlist; ++L) {
      ubase[L] = (int)units.size();
      for (int t = 0; t * R < ix->lsize[L]; ++t) units.push_back(make_int2(L, t));
      ix->rt_maxtiles = std::max(ix->rt_maxtiles, (ix->lsize[L] + R - 1) / R);
    }
    ix->rt_nunits = (int)units.size();
    ok = dalloc((void**)&ix->rt_units, units.size() * 8) &&
         cudaMemcpy(ix->rt_units, units.data(), units.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
         dalloc((void**)&ix->rt_ubase, (size_t)nlist * 4) &&
         cudaMemcpy(ix->rt_ubase, ubase.data(), (size_t)nlist * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  }
  cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  cudaDeviceGetAttribute(&ix->l2_bytes, cudaDevAttrL2CacheSize, cuda_device);
  if (ok && kind == BBC_KIND_PQ) {
    // chunk-major copy of the codes for the replicated-LUT scan (layout: k_transpose_codes)
    std::vector<long long> tb(nlist, 0);
    long long tot = 0;
    const long long gbytes = ix->nbits == 4 ? 16LL * M : 32LL * M;   // bytes per 32-object group
    for (int L = 0; L < nlist; ++L) {
      tb[L] = tot;
      tot += (long long)((ix->lsize[L] + 31) / 32) * gbytes;
    }
    ix->ct_bytes = tot;
    ok = dalloc((void**)&ix->codes_t, (size_t)tot + kCodesTailPad) &&
         dalloc((void**)&ix->tbase, (size_t)nlist * 8) &&
         cudaMemcpy(ix->tbase, tb.data(), (size_t)nlist * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemset(ix->codes_t, 0, (size_t)tot + kCodesTailPad) == cudaSuccess;
    if (ok && ix->n_local > 0) {
      if (ix->nbits == 4)
        k_pack_codes4<<<nlist, 256>>>(ix->codes, ix->loff, ix->tbase, M, ix->codes_t);
      else
        k_transpose_codes<<<(unsigned)((ix->n_local + 255) / 256), 256>>>(
            ix->codes, ix->loff, ix->tbase, nlist, ix->n_local, M, ix->codes_t);
      ok = cudaDeviceSynchronize() == cudaSuccess;
    }
  }
  if (!ok) {
    cudaError_t e = cudaGetLastError();
    return fail_load(e == cudaErrorMemoryAllocation ? BBC_ERR_OOM : BBC_ERR_IO,
                     std::string("load failed: ") + cudaGetErrorString(e));
  }
  fclose(f);
  *out = ix;
  return BBC_OK;
}

void ivf_free(bbc_index ix) {
  if (!ix) return;
  cudaSetDevice(ix->device);
  void* ptrs[] = {ix->centroids, ix->loff, ix->gsize_d, ix->ids, ix->books, ix->codes, ix->P,
                  ix->wL, ix->bits, ix->factors, ix->raw, ix->stats, ix->codes_t, ix->tbase,
                  ix->cmu, ix->cnorm, ix->rbq_tiles, ix->rbq_pc, ix->lrank, ix->pb_hi, ix->pb_lo,
                  ix->nccl_scratch, ix->rt_units, ix->rt_ubase};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& t : ix->timers) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  if (ix->nccl_x) ncclCommDestroy((ncclComm_t)ix->nccl_x);
  if (ix->nccl) ncclCommDestroy((ncclComm_t)ix->nccl);
  if (ix->h_tot) cudaFreeHost(ix->h_tot);
  for (auto e : ix->pool) cudaEventDestroy(e);
  if (ix->copy_stream) cudaStreamDestroy(ix->copy_stream);
  if (ix->copy_stream2) cudaStreamDestroy(ix->copy_stream2);
  for (int i = 0; i < 2; ++i)
    if (ix->ev_copied2[i]) cudaEventDestroy(ix->ev_copied2[i]);
  for (int i = 0; i < 2; ++i) {
    if (ix->ev_done[i]) cudaEventDestroy(ix->ev_done[i]);
    if (ix->ev_copied[i]) cudaEventDestroy(ix->ev_copied[i]);
  }
  delete ix;
}

bbc_status bbc_set_probe_mode(bbc_index ix, int32_t mode) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (mode != BBC_PROBE_SIMT && mode != BBC_PROBE_TENSOR && mode != BBC_PROBE_AUTO)
    return fail(BBC_ERR_ARG, "unknown probe mode");
  if (mode == BBC_PROBE_TENSOR && !ix->probe_tc_ok) return fail(BBC_ERR_ARG, "d too large for the tensor-core probe");
  ix->probe_mode = mode;
  return BBC_OK;
}

bbc_status bbc_set_buckets(bbc_index ix, int32_t nbuckets) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (nbuckets < 1 || nbuckets > 255) return fail(BBC_ERR_ARG, "nbuckets must be in [1, 255]");
  ix->nbuckets = nbuckets;
  return BBC_OK;
}

bbc_status bbc_set_scan_mode(bbc_index ix, int32_t mode) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (mode != BBC_SCAN_SIMT && mode != BBC_SCAN_TENSOR) return fail(BBC_ERR_ARG, "unknown scan mode");
  if (mode == BBC_SCAN_TENSOR && ix->kind == BBC_KIND_RABITQ && !ix->rbq_pc)
    return fail(BBC_ERR_ARG, "tensor-core RaBitQ scan unavailable for this index (D > 1024)");
  ix->rbq_tc = (mode == BBC_SCAN_TENSOR && ix->kind == BBC_KIND_RABITQ) ? 1 : 0;
  return BBC_OK;
}

bbc_status bbc_set_bound_rerank(bbc_index ix, int32_t on, float eps0) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (on != BBC_ALG3_OFF && on != BBC_ALG3_LIST && on != BBC_ALG3_QUERY)
    return fail(BBC_ERR_ARG, "mode must be BBC_ALG3_OFF, BBC_ALG3_LIST or BBC_ALG3_QUERY");
  if (on && ix->kind != BBC_KIND_RABITQ) return fail(BBC_ERR_ARG, "Algorithm 3 needs a RaBitQ index");
  if (on && ix->world > 1) return fail(BBC_ERR_ARG, "Algorithm 3 is single-shard only");
  if (on && ix->remap_m > 0) return fail(BBC_ERR_ARG, "Algorithm 3 uses the equal-width buckets (remap off)");
  if (on && !(eps0 > 0.f && eps0 < 1e6f)) return fail(BBC_ERR_ARG, "eps0 must be in (0, 1e6)");
  ix->alg3 = on;
  if (on) ix->alg3_eps0 = eps0;
  return BBC_OK;
}

bbc_status bbc_set_early_rerank(bbc_index ix, int32_t on) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (on != 0 && on != 1) return fail(BBC_ERR_ARG, "on must be 0 or 1");
  if (on && (ix->kind != BBC_KIND_PQ || ix->nbits != 8))
    return fail(BBC_ERR_ARG, "Algorithm 4 needs an IVF+PQ index with 8-bit codes");
  if (on && ix->world > 1) return fail(BBC_ERR_ARG, "Algorithm 4 is single-shard only");
  if (on && ix->remap_m > 0) return fail(BBC_ERR_ARG, "Algorithm 4 uses the equal-width buckets (remap off)");
  if (on && (ix->raw_u8 ? ix->d : 4 * ix->d) % 16 != 0) return fail(BBC_ERR_ARG, "Algorithm 4 needs rows of a multiple of 16 bytes");
  ix->early = on;
  return BBC_OK;
}

bbc_status bbc_set_remap(bbc_index ix, int32_t m) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (m < 0 || m > 255) return fail(BBC_ERR_ARG, "m must be 0 (off) or in [1, 255]");
  if (m > 0 && ix->early) return fail(BBC_ERR_ARG, "the equal-depth remap is off under Algorithm 4");
  if (m > 0 && ix->world > 1) return fail(BBC_ERR_ARG, "the equal-depth remap is single-shard only");
  if (m > 0 && ix->alg3) return fail(BBC_ERR_ARG, "the equal-depth remap is off under Algorithm 3");
  ix->remap_m = m;
  return BBC_OK;
}

bbc_status bbc_set_code_loads(bbc_index ix, int32_t mode) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (mode != BBC_CODES_AUTO && mode != BBC_CODES_CACHED && mode != BBC_CODES_STREAM)
    return fail(BBC_ERR_ARG, "unknown code-load mode");
  ix->code_loads = mode;
  return BBC_OK;
}

bbc_status bbc_set_scan_order(bbc_index ix, int32_t order) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (order != BBC_ORDER_AUTO && order != BBC_ORDER_PROBE && order != BBC_ORDER_SWEEP)
    return fail(BBC_ERR_ARG, "unknown scan order");
  ix->scan_order = order;
  return BBC_OK;
}

bbc_status bbc_set_rerank_order(bbc_index ix, int32_t order) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  if (order != BBC_RERANK_QUERY && order != BBC_RERANK_LIST && order != BBC_RERANK_AUTO &&
      order != BBC_RERANK_TILE)
    return fail(BBC_ERR_ARG, "unknown re-rank order");
  if (order == BBC_RERANK_TILE && !ix->rt_units)
    return fail(BBC_ERR_ARG, "the shared-memory re-rank needs fp32 rows of 128, 256, 384 or 512 bytes");
  ix->rerank_order = order;
  return BBC_OK;
}

bbc_status bbc_index_info(bbc_index ix, bbc_index_info_t* info) {
  if (!ix || !info) return fail(BBC_ERR_ARG, "null argument");
  info->n = ix->N; info->d = ix->d; info->nlist = ix->nlist; info->kind = ix->kind;
  info->m = ix->M; info->dpad = ix->D; info->raw_u8 = ix->raw_u8; info->n_local = ix->n_local;
  info->max_list = ix->max_list; info->rank = ix->rank; info->world = ix->world;
  info->metric = ix->metric;
  info->nbits = ix->kind == BBC_KIND_PQ ? ix->nbits : 1;
  return BBC_OK;
}

bbc_status bbc_workspace_size(bbc_index ix, int64_t nq, int32_t k, int32_t nprobe, int64_t budget,
                              size_t* bytes, size_t* min_bytes) {
  if (!ix || !bytes) return fail(BBC_ERR_ARG, "null argument");
  if (nprobe < 1 || nprobe > ix->nlist || k < 1 || nq < 0 || budget < k)
    return fail(BBC_ERR_ARG, "bad arguments");
  Plan p = make_plan(ix, nprobe, k, ix->world, ix->world > 1 || ix->force_dist);
  *bytes = p.fixed + (size_t)std::max<int64_t>(nq, 1) * p.per_query;
  if (min_bytes) *min_bytes = p.fixed + p.per_query;
  return BBC_OK;
}

bbc_status bbc_query_capacity(bbc_index ix, int32_t nprobe, int64_t* cap) {
  if (!ix || !cap) return fail(BBC_ERR_ARG, "null argument");
  if (nprobe < 1 || nprobe > ix->nlist) return fail(BBC_ERR_ARG, "bad nprobe");
  *cap = make_plan(ix, nprobe, 1).cap;
  return BBC_OK;
}

bbc_status bbc_search(bbc_index ix, const float* queries, int64_t nq, int32_t k, int32_t nprobe,
                      int64_t budget, int64_t* out_ids, float* out_d2, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return run_one(ix, queries, nq, k, nprobe, budget, out_ids, out_d2, workspace,
                 workspace_bytes, stream, false, nullptr);
}

bbc_status bbc_search_host(bbc_index ix, const float* queries_host, int64_t nq, int32_t k,
                           int32_t nprobe, int64_t budget, int64_t* out_ids_host,
                           float* out_d2_host, void* workspace, size_t workspace_bytes,
                           void* stream) {
  return run_one(ix, queries_host, nq, k, nprobe, budget, out_ids_host, out_d2_host, workspace,
                 workspace_bytes, stream, true, nullptr);
}

bbc_status bbc_search_debug(bbc_index ix, const float* queries, int64_t nq, int32_t k,
                            int32_t nprobe, int64_t budget, int64_t* out_ids, float* out_d2,
                            void* workspace, size_t workspace_bytes, void* stream,
                            const bbc_debug_bufs* dbg) {
  if (!dbg) return fail(BBC_ERR_ARG, "null debug buffers");
  return run_one(ix, queries, nq, k, nprobe, budget, out_ids, out_d2, workspace,
                 workspace_bytes, stream, false, dbg);
}

bbc_status bbc_search_group(const bbc_index* shards, int nshards, const float* queries, int64_t nq,
                            int32_t k, int32_t nprobe, int64_t budget, int64_t* out_ids,
                            float* out_d2, void* const* workspaces, const size_t* workspace_bytes,
                            void* stream) {
  if (!shards || !workspaces || !workspace_bytes || nshards < 1 || nshards > 8)
    return fail(BBC_ERR_ARG, "bbc_search_group: 1..8 shards with workspaces");
  std::vector<Shard> sh(nshards);
  for (int i = 0; i < nshards; ++i) {
    bbc_index_s* ix = shards[i];
    if (!ix) return fail(BBC_ERR_ARG, "null shard");
    if (ix->world != nshards || ix->rank != i || ix->device != shards[0]->device)
      return fail(BBC_ERR_ARG, "shard i must be loaded with rank i, world nshards, same device");
    sh[i].ix = ix;
    sh[i].ws = (char*)workspaces[i];
    sh[i].ws_bytes = workspace_bytes[i];
    sh[i].rank = i;
  }
  GroupComm c(nshards);
  return run(sh, &c, queries, nq, k, nprobe, budget, out_ids, out_d2, stream, false, nullptr);
}

bbc_status bbc_nccl_unique_id(void* id128) {
  if (!id128) return fail(BBC_ERR_ARG, "null argument");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(BBC_ERR_NCCL, "ncclGetUniqueId failed");
  memcpy(id128, &id, sizeof(id));
  return BBC_OK;
}

bbc_status bbc_comm_init(bbc_index ix, const void* id128, int rank, int world) {
  if (!ix || !id128) return fail(BBC_ERR_ARG, "null argument");
  if (rank != ix->rank || world != ix->world)
    return fail(BBC_ERR_ARG, "rank/world must match the shard the index was loaded as");
  if (cudaSetDevice(ix->device) != cudaSuccess) return fail(BBC_ERR_CUDA, "cudaSetDevice");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  const ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) return fail(BBC_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  ncclComm_t cx;                      // the result all-gather's own communicator (copy stream)
  const ncclResult_t r2 = ncclCommSplit(c, 0, rank, &cx, nullptr);
  if (r2 != ncclSuccess) {
    ncclCommDestroy(c);
    return fail(BBC_ERR_NCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r2));
  }
  if (ix->nccl_x) ncclCommDestroy((ncclComm_t)ix->nccl_x);
  if (ix->nccl) ncclCommDestroy((ncclComm_t)ix->nccl);
  ix->nccl = (void*)c;
  ix->nccl_x = (void*)cx;
  if (!ix->nccl_scratch && cudaMalloc((void**)&ix->nccl_scratch, 8) != cudaSuccess)
    return fail(BBC_ERR_CUDA, "cudaMalloc (communicator scratch)");
  ix->force_dist = world == 1;
  return BBC_OK;
}

bbc_status bbc_set_timing(bbc_index ix, int enable) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  ix->timing = enable != 0;
  return BBC_OK;
}

bbc_status bbc_get_timing(bbc_index ix, float* ms, int n, int64_t* calls) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  for (auto& t : ix->timers) {
    cudaEventSynchronize(t.b);
    float e = 0.f;
    cudaEventElapsedTime(&e, t.a, t.b);
    ix->stage_ms[t.stage] += e;
    ix->pool.push_back(t.a);
    ix->pool.push_back(t.b);
  }
  ix->timers.clear();
  for (int i = 0; i < n && i < BBC_NUM_STAGES; ++i) ms[i] = (float)ix->stage_ms[i];
  if (calls) *calls = ix->timed_calls;
  for (double& v : ix->stage_ms) v = 0;
  ix->timed_calls = 0;
  return BBC_OK;
}

bbc_status bbc_last_stats(bbc_index ix, int64_t* probed, int64_t* candidates, int64_t* micro) {
  return bbc_last_stats2(ix, probed, candidates, micro, nullptr);
}

bbc_status bbc_last_stats2(bbc_index ix, int64_t* probed, int64_t* candidates, int64_t* micro,
                           int64_t* sampled) {
  if (!ix) return fail(BBC_ERR_ARG, "null index");
  long long h[4];
  CU(cudaMemcpy(h, ix->stats, sizeof(h), cudaMemcpyDeviceToHost));
  if (probed) *probed = h[0];
  if (candidates) *candidates = h[1];
  if (micro) *micro = ix->microbatches;
  if (sampled) *sampled = h[2];
  return BBC_OK;
}

bbc_status bbc_stats_vector(bbc_index ix, int64_t* out, int32_t n) {
  if (!ix || (!out && n > 0) || n < 0) return fail(BBC_ERR_ARG, "bad argument");
  long long h[kNStats];
  CU(cudaMemcpy(h, ix->stats, sizeof(h), cudaMemcpyDeviceToHost));
  const long long v[9] = {h[0], h[1], h[2], h[3], ix->microbatches, ix->rr_list_batches, h[4], h[5], h[6]};
  for (int i = 0; i < n && i < 9; ++i) out[i] = v[i];
  return BBC_OK;
}

}  // extern "C"
