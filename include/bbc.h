/*
 * bbc.h -- C ABI of libbbc.so: the B200 query hot path of BBC, the bucket-based result
 * collector for large-k ANN search over quantized IVF indexes (arXiv 2604.01960).
 *
 * "P:Lnnn" cites a line of the paper text; DESIGN.md section 2 lists the readings.
 *
 * One call, bbc_search(), runs the whole path for a batch of queries (BASELINE.json north_star):
 *   a1 coarse probe -- the nprobe nearest IVF lists, nearest first
 *   a2 query tables -- PQ LUT / RaBitQ rotated + 4-bit query code
 *   a3 sample       -- estimates of the nearest lists; d_min, d_max
 *   a4 Push         -- estimate + bucket id of every probed object, histogram (Alg. 1 l.1-4,
 *                      Eq. 6)
 *   a5 Update       -- threshold bucket tau: first cumulative count >= budget (Alg. 1 l.5-11)
 *   a6 Collect      -- candidate superset S* = objects in buckets <= tau
 *   a7 re-rank      -- exact squared L2 of every candidate against raw vectors
 *   a8 select       -- the k candidates with the smallest (exact d^2, id)
 *
 * Conventions
 *   - All "device" pointers are CUDA device memory of the device the index was loaded on; all
 *     "host" pointers are ordinary (or pinned) host memory.  No function allocates device memory
 *     except ivf_load (index arrays, freed by ivf_free).  Scratch lives in the caller's workspace.
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and the search
 *     functions return after enqueueing (bbc_search_host synchronises the stream before it
 *     returns).  One search may be in flight per workspace.
 *   - Distances are squared Euclidean.  Output ids are the original row ids of the database.
 *   - Errors: every function returns BBC_OK or an error code and then nothing was enqueued
 *     (argument errors) or the stream state is unspecified (CUDA errors; the index handle
 *     becomes unusable: later calls return BBC_ERR_STATE).  bbc_last_error() gives a message.
 */
#ifndef BBC_H_
#define BBC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bbc_index_s* bbc_index;

typedef enum {
  BBC_OK = 0,
  BBC_ERR_ARG = 1,     /* invalid argument (k, nprobe, budget, nq, null pointer, workspace size) */
  BBC_ERR_IO = 2,      /* index file cannot be opened or read                                    */
  BBC_ERR_FORMAT = 3,  /* index file malformed (magic, version, section sizes)                    */
  BBC_ERR_CUDA = 4,    /* a CUDA runtime error (message in bbc_last_error)                        */
  BBC_ERR_NCCL = 5,    /* a collective failed (multi-GPU)                                         */
  BBC_ERR_OOM = 6,     /* device allocation in ivf_load failed                                    */
  BBC_ERR_STATE = 7    /* handle unusable after an earlier CUDA/NCCL error                        */
} bbc_status;

/* Index kinds (file header field `kind`). */
#define BBC_KIND_PQ 1      /* 8-bit product quantization, M sub-quantizers of 256 codewords   */
#define BBC_KIND_RABITQ 2  /* 1-bit RaBitQ codes over a random rotation, factors (r_o, g_o)  */
/* Metric of an index (header field 11).  Every distance the library handles is a key where
 * smaller is better: squared L2, or for inner product the negated similarity -<q, x> (the
 * result buffer "applies to ... cosine similarity and inner product"; cosine =
 * inner product of unit-norm vectors).  IP is supported for PQ indexes (BBC_ERR_FORMAT for
 * RaBitQ); its out_d2 holds -<q, x>. */
#define BBC_METRIC_L2 0
#define BBC_METRIC_IP 1

/*
 * ivf_load -- read a BBCIVF01 index file (layout: DESIGN.md section 4 / datagen/index_file.py):
 *   bytes [0,8) magic "BBCIVF01"; [8,256) 31 x int64 header {version=1, kind, raw_dtype(0 f32,
 *   1 u8), N, d, nlist, M, nbits, D, seed, n_sections=10}; [256,416) section table of
 *   (int64 offset, int64 nbytes); sections centroids f32[nlist*d], list_offsets i64[nlist+1],
 *   ids i64[N], codebooks f32[M*256*(d/M)], codes u8[N*M], P f32[D*D], wL f32[nlist*D],
 *   bits u8[N*D/8], factors f32[N*2], raw f32|u8[N*d]; per-object arrays in list order.
 * and upload it to `cuda_device`.  N must be < 2^31 (BBC_ERR_FORMAT otherwise): the kernels
 * carry rows and original ids as 32-bit integers (the ids file section and out_ids stay int64;
 * ids are widened on output).  With world > 1 only the lists assigned to `rank` are kept
 * (lists sorted by (size desc, id asc) and given greedily to the least-loaded rank); centroids,
 * codebooks, rotation and every list's size are replicated.  On success *out owns the device
 * arrays until ivf_free.
 */
bbc_status ivf_load(const char* path, int rank, int world, int cuda_device, bbc_index* out);
void ivf_free(bbc_index index);

typedef struct {
  int64_t n;           /* database size N (all ranks)                  */
  int32_t d;           /* dimensionality                               */
  int32_t nlist;       /* IVF lists                                    */
  int32_t kind;        /* BBC_KIND_PQ or BBC_KIND_RABITQ               */
  int32_t m;           /* PQ sub-quantizers (0 for RaBitQ)             */
  int32_t dpad;        /* RaBitQ padded dimension D (0 for PQ)         */
  int32_t raw_u8;      /* 1 if raw vectors are uint8, 0 if fp32         */
  int64_t n_local;     /* objects held by this rank                    */
  int32_t max_list;    /* largest list size                            */
  int32_t rank, world; /* shard of this handle                         */
  int32_t metric;      /* BBC_METRIC_L2 or BBC_METRIC_IP               */
  int32_t nbits;       /* PQ code bits (8 or 4); 1 for RaBitQ          */
} bbc_index_info_t;

bbc_status bbc_index_info(bbc_index index, bbc_index_info_t* info);

/*
 * bbc_set_probe_mode -- how step a1 (coarse probe, route P:L392; nearest-first order P:L1146)
 * computes the nprobe nearest lists.  All modes return the same lists: the nprobe smallest
 * (canonical fp32 d^2, list id) keys.
 *   BBC_PROBE_SIMT   : canonical fp32 d^2 of every (query, centroid) on the CUDA cores.
 *   BBC_PROBE_TENSOR : (d <= 1024) the tensor cores (tcgen05, kind::tf32, 3xTF32 split)
 *                      compute d~ with a proven error bound; the shortlist that provably holds
 *                      the nprobe nearest lists is re-scored canonically.
 *   BBC_PROBE_AUTO   : (default) TENSOR when available and nprobe <= nlist / 16 (the re-score
 *                      reads nprobe centroid rows per query), SIMT otherwise.
 * Errors: BBC_ERR_ARG for a null index, an unknown mode, or TENSOR with d > 1024.  The mode is
 * per handle; it must not change while a search on the handle is in flight.
 */
#define BBC_PROBE_SIMT 0
#define BBC_PROBE_TENSOR 1
#define BBC_PROBE_AUTO 2
bbc_status bbc_set_probe_mode(bbc_index index, int32_t mode);

/*
 * bbc_set_scan_mode -- how steps a3/a4 compute RaBitQ estimated distances (B_q = 4, P:L1440;
 * estimator DESIGN.md 2.2).  Both modes give bit-identical estimates (the code/query inner
 * product is an exact integer either way).  PQ indexes ignore the mode (replicated-LUT scan).
 *   BBC_SCAN_SIMT   : per (query, list) CTA, 4 popcounts per 32 code bits.
 *   BBC_SCAN_TENSOR : (default, D <= 1024) list-major: the codes of a list times the 4-bit
 *                     query codes of every query probing it, one integer GEMM on the tensor
 *                     cores (tcgen05 kind::i8) per 128-object tile.
 * Errors: BBC_ERR_ARG for a null index, an unknown mode, or TENSOR on a RaBitQ index with
 * D > 1024.  Must not change while a search on the handle is in flight.
 */
/*
 * bbc_set_buckets -- B, the number of regular equal-width buckets of the result buffer over
 * [d_min, d_max] (Eq. 6; the paper's m, Eq. 3 and Table 4).  Default
 * 255 (8-bit bucket ids; id 255 = beyond d_max, never a candidate).  Fewer buckets give a
 * coarser threshold and a larger candidate superset S*.  BBC_ERR_ARG unless 1 <= B <= 255.
 */
bbc_status bbc_set_buckets(bbc_index index, int32_t nbuckets);

/*
 * bbc_set_remap -- the n_ew -> m equal-depth remap of the result buffer ("first computes
 * n_ew equal-width buckets and then reassigns these buckets into m equal-depth buckets, where a
 * lookup table map is used"; Eq. 6 with map; reading R6).  m = 0 (default):
 * the equal-width cells are the buckets.  m in [1, 255]: per query, the sample's histogram over
 * the cells defines m equal-depth buckets (greedy: a bucket closes at the first cell where the
 * running sample count reaches its share); the threshold is the first bucket whose count reaches
 * the budget, and S* is every object whose bucket is at or below it -- a superset of the
 * equal-width S*.  BBC_ERR_ARG for m outside [0, 255] or m > 0 on a sharded handle.
 */
bbc_status bbc_set_remap(bbc_index index, int32_t m);

/*
 * bbc_set_bound_rerank -- Algorithm 3, the bound-aware re-rank of IVF+RaBitQ (
 * SURVEY 8(f) f1; reading R21), in place of steps a4..a7 of a RaBitQ search.  mode
 * BBC_ALG3_LIST or BBC_ALG3_QUERY (same results; how the exact distances are gathered, below):
 * every probed object's estimate gets the RaBitQ bound lb/ub = est -/+ ((2 r_o) r)(t_o eps),
 * t_o = sqrt(1 - g_o^2)/g_o, eps = eps0/sqrt(D - 1) (eps0 = 1.9 in the paper,
 * P:L1440), both bucketed with the sample's codebook (Eq. 6); tau = the first bucket where the
 * upper-bound counts reach k; objects with a_lb <= tau are the candidates; the marginal-bucket
 * loop of l.12-21 re-ranks B_l[i] and B_u[j] until i >= j, then B_u[j]'s leftovers (l.22); the
 * result is the k smallest (exact d^2, id) of the re-ranked objects.  bbc_search_debug reports
 * the upper-bound histogram in `hist`, tau, the candidates (a_lb <= tau) in cand_ids with exact
 * d^2 for the re-ranked ones and +inf for the others.  `budget` still sizes the sample (R5).
 * BBC_ALG3_LIST computes the exact d^2 of every candidate (a_lb <= tau) with the list-order
 * re-rank (rows shared through L2) and runs the loop on those distances; BBC_ALG3_QUERY gathers
 * only B_exact's rows, one CTA per query as the loop reaches them (fewer rows, slower on the GPU,
 * DESIGN.md 8).  The rows gathered are counted in bbc_last_stats' candidates.
 * BBC_ALG3_OFF (default): Algorithm 1's superset.  The workspace grows by up to 12 bytes per
 * probed-object slot per query (query the size after the change).  BBC_ERR_ARG for a PQ index,
 * a sharded handle, an active remap, an unknown mode or eps0 outside (0, 1e6); the sharded path
 * (bbc_search_group, world > 1) returns BBC_ERR_ARG while it is on.
 */
#define BBC_ALG3_OFF 0
#define BBC_ALG3_LIST 1
#define BBC_ALG3_QUERY 2
bbc_status bbc_set_bound_rerank(bbc_index index, int32_t mode, float eps0);

/*
 * bbc_set_early_rerank -- Algorithm 4, the early re-ranking of IVF+PQ (SURVEY 8(f)
 * f2; reading R22).  on = 1: after the sample stage the predicted threshold bucket
 * tau_pred is the bucket of the floor(budget * |O_sample| / n_o)-th (at least the first) smallest
 * sample estimate (l.2-4); straight after the main scan pass has written the bucket
 * ids -- before the threshold is known -- every object scanned after the sample whose bucket
 * lies below tau_pred gets its exact distance (l.9-11: "we immediately compute its exact
 * distance"; k_early_rows); the compaction hands those distances to the candidates
 * among them and the re-rank computes only the remaining candidates' (l.15).
 * Results are those of Algorithm 1 (same candidates; early distances are rounded in another
 * order, within the 1e-5 tolerance).  bbc_search_debug reports tau_pred and, per candidate,
 * whether its distance was computed early; bbc_stats_vector entries 7 and 8 count the objects
 * given an early distance and the candidates that used one.  The workspace grows by 4 bytes per
 * probed-object slot per query (query the size after the change).  on = 0 (default): Algorithm 1.
 * BBC_ERR_ARG for a RaBitQ or 4-bit PQ index, a sharded handle, an active remap or another
 * value of on; the sharded paths (bbc_search_group, world > 1) return BBC_ERR_ARG while it is on.
 */
bbc_status bbc_set_early_rerank(bbc_index index, int32_t on);

#define BBC_SCAN_SIMT 0
#define BBC_SCAN_TENSOR 1
bbc_status bbc_set_scan_mode(bbc_index index, int32_t mode);

/*
 * bbc_set_rerank_order -- the work order of step a7, the exact re-rank of S* (P:L413).
 * Results are identical in both orders (each candidate's distance is computed by the same lanes
 * in the same arithmetic order); only which rows are read together differs.
 *   BBC_RERANK_QUERY : CTAs walk one query's candidates (rows of one query in flight).
 *   BBC_RERANK_LIST  : the run of candidates a query has in one inverted list is a segment;
 *                      segments are ordered by list, so the rows in flight belong to a few
 *                      lists shared by every query probing them and are served from L2.
 *   BBC_RERANK_TILE  : list order with each list's rows staged in shared memory, one tile of
 *                      consecutive rows per CTA by a bulk copy, every candidate of every query in
 *                      that tile computed from shared memory (fp32 rows of 128, 256, 384 or 512
 *                      bytes; BBC_ERR_ARG otherwise).  Measured slower than LIST.
 *   BBC_RERANK_AUTO  : (default) LIST when the micro-batch re-ranks each row >= 4 times on
 *                      average (nq * budget / N), else QUERY.
 * BBC_ERR_ARG for a null index or an unknown order.  Must not change while a search on the
 * handle is in flight.
 */
#define BBC_RERANK_QUERY 0
#define BBC_RERANK_LIST 1
#define BBC_RERANK_AUTO 2
#define BBC_RERANK_TILE 3
bbc_status bbc_set_rerank_order(bbc_index index, int32_t order);

/*
 * bbc_set_code_loads -- the L1 policy of the 8-bit PQ scan's 16-byte code loads (step a4).  Same
 * results in every mode; only the cache behaviour differs.
 *   BBC_CODES_CACHED : ld.global.nc through L1 (best when the codes are L2-resident).
 *   BBC_CODES_STREAM : ld.global.nc.L1::no_allocate (codes streamed once from HBM only evict L1).
 *   BBC_CODES_AUTO   : (default) STREAM when this shard's codes exceed half of the L2 size the
 *                      device reports (cudaDevAttrL2CacheSize), CACHED otherwise.
 * BBC_ERR_ARG for a null index or an unknown mode.  Must not change while a search is in flight.
 */
#define BBC_CODES_AUTO 0
#define BBC_CODES_CACHED 1
#define BBC_CODES_STREAM 2
bbc_status bbc_set_code_loads(bbc_index index, int32_t mode);

/*
 * bbc_set_scan_order -- the order in which the 8-bit PQ scan (steps a3/a4) visits the probed
 * objects.  Same results in every order (each object's estimate and bucket id go to its
 * probe-order position; the histogram is an integer sum); only the L2 reuse of the codes differs.
 *   BBC_ORDER_PROBE : query after query, each query's lists nearest first (probe order).
 *   BBC_ORDER_SWEEP : each query's lists by ascending list id, work items issued by the list
 *                    holding their first object, so the items in flight share a window of lists
 *                    whose codes stay in L2 (a list's codes come from HBM about once per pass);
 *                    and the sample pass fills its last work item with the lists that follow the
 *                    sample in probe order (their bucket ids come from those estimates).
 *   BBC_ORDER_AUTO  : (default) SWEEP when this shard's codes exceed half of the L2 size, PROBE
 *                    otherwise.
 * BBC_ERR_ARG for a null index or an unknown order.  Must not change while a search is in flight.
 */
#define BBC_ORDER_AUTO 0
#define BBC_ORDER_PROBE 1
#define BBC_ORDER_SWEEP 2
bbc_status bbc_set_scan_order(bbc_index index, int32_t order);

/*
 * bbc_workspace_size -- bytes of device workspace bbc_search needs for (nq, k, nprobe, budget).
 * The workspace holds per-query scratch sized for the nprobe largest lists (cell ids, candidate
 * rows and distances) plus query/output staging used by bbc_search_host.  Queries are processed
 * in micro-batches that fit; a larger workspace means larger micro-batches.  `min_bytes` (may be
 * NULL) receives the smallest workspace that still works (one query per micro-batch).
 */
bbc_status bbc_workspace_size(bbc_index index, int64_t nq, int32_t k, int32_t nprobe,
                              int64_t budget, size_t* bytes, size_t* min_bytes);

/*
 * bbc_query_capacity -- upper bound on the objects one query probes on this shard (and hence on
 * |S*|): the sum of the nprobe largest local lists.  Sizes the per-query debug buffers.
 */
bbc_status bbc_query_capacity(bbc_index index, int32_t nprobe, int64_t* cap);

/*
 * bbc_search -- top-k of every query (device pointers).
 *   queries  device f32 [nq x d], row-major (uint8-valued queries for a uint8 index are passed
 *            as fp32)
 *   k        1 <= k <= N                        (else BBC_ERR_ARG)
 *   nprobe   1 <= nprobe <= nlist               (else BBC_ERR_ARG)
 *   budget   candidate budget, budget >= k      (else BBC_ERR_ARG); budget >= probed count means
 *            every probed object is re-ranked (tau = infinity, Alg. 1 l.11)
 *   out_ids  device i64 [nq x k]; out_d2 device f32 [nq x k].  Row i holds the k probed
 *            candidates with the smallest (exact d^2, id), in candidate (probe) order, not sorted.
 *            (Under bbc_set_bound_rerank the candidate order, and so this order, is unspecified.)
 *            When fewer than k objects are probed the row is padded with (id -1, d^2 +inf).
 *   workspace/workspace_bytes: device scratch of at least the `min_bytes` of bbc_workspace_size.
 *   stream   cudaStream_t (void*), NULL = default stream.
 * On an unsharded handle without stage timing the call only enqueues stream-ordered work (no
 * host synchronisation, no allocation), so it can be captured into a CUDA graph and replayed
 * (tests/test_gpu_parity.py::test_search_captures_into_a_cuda_graph).
 */
bbc_status bbc_search(bbc_index index, const float* queries, int64_t nq, int32_t k,
                      int32_t nprobe, int64_t budget, int64_t* out_ids, float* out_d2,
                      void* workspace, size_t workspace_bytes, void* stream);

/*
 * bbc_search_host -- same as bbc_search, but queries/out_ids/out_d2 are HOST pointers.  The
 * host->device copy of the queries, the search and the device->host copy of the results are
 * enqueued on `stream` (staging buffers come from the workspace, which must be at least the
 * `bytes` of bbc_workspace_size for this nq), then the stream is synchronised.
 */
bbc_status bbc_search_host(bbc_index index, const float* queries_host, int64_t nq, int32_t k,
                           int32_t nprobe, int64_t budget, int64_t* out_ids_host,
                           float* out_d2_host, void* workspace, size_t workspace_bytes,
                           void* stream);

/*
 * Intermediates for parity tests.  Device pointers, any may be NULL; per-query strides are the
 * `*_stride` values the caller passes (elements).  Requires a workspace in which all nq queries
 * fit in one micro-batch (workspace_bytes >= bbc_workspace_size(...).bytes).
 *   probe   i32 [nq x nprobe]  lists, nearest first          rq2    f32 [nq x nprobe]
 *   nsample i32 [nq]           sample lists s (0 = tau inf)  edges  f32 [nq x 2] (d_min, d_max)
 *   hist    i32 [nq x 256]     bucket histogram (255 = overflow, not counted)
 *   tau     i32 [nq]           threshold bucket (1<<30 = infinity)
 *   n_probed i32 [nq]          objects probed (n_o)
 *   est     f32 [nq x est_stride]  estimated distances in probe order (only when non-NULL;
 *                                  costs an extra pass)
 *   n_cand  i32 [nq]           |S*|
 *   cand_ids i64 [nq x cand_stride]  ids of S* in probe order
 *   cand_d2  f32 [nq x cand_stride]  exact d^2 of S*
 *   tau_pred i32 [nq]          Algorithm 4's predicted threshold bucket (0 when it is off)
 *   cand_early u8 [nq x cand_stride]  1 if the candidate's d^2 was computed early (Algorithm 4)
 * (the last two may be NULL)
 */
typedef struct {
  int32_t* probe;
  float* rq2;
  int32_t* nsample;
  float* edges;
  int32_t* hist;
  int32_t* tau;
  int32_t* n_probed;
  float* est;
  int64_t est_stride;
  int32_t* n_cand;
  int64_t* cand_ids;
  float* cand_d2;
  int64_t cand_stride;
  int32_t* tau_pred;
  uint8_t* cand_early;
} bbc_debug_bufs;

bbc_status bbc_search_debug(bbc_index index, const float* queries, int64_t nq, int32_t k,
                            int32_t nprobe, int64_t budget, int64_t* out_ids, float* out_d2,
                            void* workspace, size_t workspace_bytes, void* stream,
                            const bbc_debug_bufs* dbg);

/*
 * Multi-GPU (database sharded by IVF list).  Each rank loads its shard with
 * ivf_load(path, rank, world, device), rank 0 creates an NCCL id with bbc_nccl_unique_id and
 * broadcasts the 128 bytes (e.g. through torch.distributed), every rank calls bbc_comm_init, then
 * every rank calls bbc_search with the SAME queries and parameters (SPMD).  The exchange steps
 * (sample minimum and budget-th estimate, bucket histogram, final top-k) are NCCL all-reduces
 * enqueued on the search stream; every rank receives the full result (replicated).  Results are
 * identical for every world size.  Calling bbc_comm_init on a world-1 index makes bbc_search
 * take the same sharded code path with a 1-rank communicator (used by tests).
 */
bbc_status bbc_nccl_unique_id(void* id128);
bbc_status bbc_comm_init(bbc_index index, const void* id128, int rank, int world);

/*
 * bbc_search_group -- the sharded search for nshards (<= 8) shards held by ONE process on one
 * device: shard i loaded with ivf_load(path, i, nshards, device).  The exchange steps are
 * element-wise reductions across the shards' workspaces on `stream` (no NCCL); used to test the
 * sharded algebra on a single GPU.  workspaces[i] / workspace_bytes[i]: per-shard device scratch
 * (bbc_workspace_size of shard i).  out_ids/out_d2: device, [nq x k].
 */
bbc_status bbc_search_group(const bbc_index* shards, int nshards, const float* queries, int64_t nq,
                            int32_t k, int32_t nprobe, int64_t budget, int64_t* out_ids,
                            float* out_d2, void* const* workspaces, const size_t* workspace_bytes,
                            void* stream);

/*
 * Stage timing: when enabled, bbc_search records CUDA events on `stream` around each kernel of
 * the path; bbc_get_timing returns the summed milliseconds per stage of the searches since the
 * last call (and resets them).  Stages: BBC_STAGE_* below.  Synchronises the stream.
 */
enum {
  BBC_STAGE_PROBE = 0,   /* a1: coarse distances + nprobe selection */
  BBC_STAGE_TABLES = 1,  /* a2: LUT / rotation                      */
  BBC_STAGE_SAMPLE = 2,  /* a3: sample estimates + edge selection (+ the sample objects' bucket ids) */
  BBC_STAGE_SCAN = 3,    /* a4: Push of the other probed objects (code scan + histogram)           */
  BBC_STAGE_COMPACT = 4, /* a5+a6: threshold + superset compaction  */
  BBC_STAGE_RERANK = 5,  /* a7: exact re-rank gather                */
  BBC_STAGE_SELECT = 6,  /* a8: final top-k                         */
  BBC_STAGE_COMM = 7,    /* a9: collectives (world > 1)             */
  BBC_NUM_STAGES = 8
};
bbc_status bbc_set_timing(bbc_index index, int enable);
bbc_status bbc_get_timing(bbc_index index, float* ms, int n, int64_t* calls);

/* Per-search counters of the last bbc_search on this handle (host copy; synchronises the
 * stream): total probed objects (sum of n_o), total candidates (sum of |S*|), micro-batches. */
bbc_status bbc_last_stats(bbc_index index, int64_t* probed, int64_t* candidates,
                          int64_t* microbatches);
/* Same, plus the number of sample objects estimated in step a3 (summed over queries). */
bbc_status bbc_last_stats2(bbc_index index, int64_t* probed, int64_t* candidates,
                           int64_t* microbatches, int64_t* sampled);
/* Counters of the last search, in order: probed objects, candidates |S*|, sample objects,
 * lists shortlisted by the tensor-core probe (0 in SIMT mode), micro-batches, micro-batches
 * re-ranked in list order, objects estimated by the PQ sample pass (the sample plus, in sweep
 * order, the lists that fill its last work item; 0 for RaBitQ), objects the scan gave an early
 * exact distance and candidates that used one (Algorithm 4, bbc_set_early_rerank; else 0).
 * Copies the first n (<= 9) into out (host memory).  BBC_ERR_ARG for a null index or out with n > 0. */
bbc_status bbc_stats_vector(bbc_index index, int64_t* out, int32_t n);

/* Number of CUDA kernels this library has launched in this process. */
int64_t bbc_launch_count(void);

/*
 * bbc_measure_l2_read -- measurement utility (not part of the search path): the device's L2 ->
 * SM read bandwidth in GB/s, from CTAs that each stream an L2-resident buffer of `bytes`
 * (>= 1 MiB; choose well below the L2 size) `reps` times with 16-byte loads (the best of 4, 8
 * and 16 loads in flight per thread at 4 and 8 CTAs of 256 threads per SM).  The roofline of
 * the list-order re-rank, whose rows are served from L2.  Allocates and frees its own buffer
 * on `cuda_device`.  BBC_ERR_ARG for bad sizes, BBC_ERR_CUDA on a CUDA failure.
 */
bbc_status bbc_measure_l2_read(int32_t cuda_device, size_t bytes, int32_t reps, double* gbs);

/*
 * bbc_measure_smem_lookups -- measurement utility (not part of the search path): the device's
 * shared-memory lookup rate in G lookups/s -- one CTA of 32 warps per SM, every lane reading
 * 4-byte words at conflict-free addresses (one wavefront per warp instruction, as the 8-bit PQ
 * scan's replicated LUT) and adding them into fp32 sums, `rounds` x 32 reads per thread.  The
 * roofline of the LUT lookups of the PQ scan.  BBC_ERR_ARG for rounds < 1.
 */
bbc_status bbc_measure_smem_lookups(int32_t cuda_device, int32_t rounds, double* glookups);

/* Message for the last non-OK status returned on the calling thread. */
const char* bbc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BBC_H_ */
