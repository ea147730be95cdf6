"""Python binding of libbbc.so (include/bbc.h): argument marshalling only.

Every step of the query path runs in the library's CUDA kernels.  There is no CPU fallback:
if the library cannot be loaded, or no CUDA device is present, the calls raise.

    idx = Index(path)                                   # ivf_load
    ids, d2 = idx.search(q, k, nprobe, budget)          # bbc_search (q: cuda fp32 [nq, d])
    ids, d2 = idx.search_host(q_np, k, nprobe, budget)  # bbc_search_host (numpy in, numpy out)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BBC_LIB: load a variant build instead (kernel tuning experiments)
LIB_PATH = os.environ.get("BBC_LIB") or os.path.join(_HERE, "libbbc.so")

# names exported by include/bbc.h (checked by tests/test_lib_exports.py)
EXPORTS = ("ivf_load", "ivf_free", "bbc_index_info", "bbc_workspace_size", "bbc_query_capacity",
           "bbc_search",
           "bbc_search_host", "bbc_search_debug", "bbc_set_timing", "bbc_get_timing",
           "bbc_last_stats", "bbc_launch_count", "bbc_last_error", "bbc_nccl_unique_id",
           "bbc_comm_init", "bbc_search_group", "bbc_last_stats2", "bbc_set_probe_mode",
           "bbc_set_scan_mode", "bbc_stats_vector", "bbc_set_buckets", "bbc_set_rerank_order",
           "bbc_measure_l2_read", "bbc_set_remap", "bbc_set_code_loads",
           "bbc_measure_smem_lookups", "bbc_set_scan_order", "bbc_set_bound_rerank",
           "bbc_set_early_rerank")

STAGES = ("probe", "tables", "sample", "scan", "compact", "rerank", "select", "comm")
TAU_INF = 1 << 30
KIND_PQ, KIND_RABITQ = 1, 2


class BBCError(RuntimeError):
    pass


class IndexInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int32), ("nlist", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("m", ctypes.c_int32), ("dpad", ctypes.c_int32),
                ("raw_u8", ctypes.c_int32), ("n_local", ctypes.c_int64),
                ("max_list", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("metric", ctypes.c_int32), ("nbits", ctypes.c_int32)]


class DebugBufs(ctypes.Structure):
    _fields_ = [("probe", ctypes.c_void_p), ("rq2", ctypes.c_void_p),
                ("nsample", ctypes.c_void_p), ("edges", ctypes.c_void_p),
                ("hist", ctypes.c_void_p), ("tau", ctypes.c_void_p),
                ("n_probed", ctypes.c_void_p), ("est", ctypes.c_void_p),
                ("est_stride", ctypes.c_int64), ("n_cand", ctypes.c_void_p),
                ("cand_ids", ctypes.c_void_p), ("cand_d2", ctypes.c_void_p),
                ("cand_stride", ctypes.c_int64), ("tau_pred", ctypes.c_void_p),
                ("cand_early", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """The loaded libbbc.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BBCError(f"{LIB_PATH} not built (run paper_2604_01960_b200/build.py)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.ivf_load.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(vp)]
        L.ivf_free.argtypes = [vp]
        L.ivf_free.restype = None
        L.bbc_index_info.argtypes = [vp, ctypes.POINTER(IndexInfo)]
        L.bbc_workspace_size.argtypes = [vp, i64, i32, i32, i64, ctypes.POINTER(ctypes.c_size_t),
                                         ctypes.POINTER(ctypes.c_size_t)]
        L.bbc_search.argtypes = [vp, vp, i64, i32, i32, i64, vp, vp, vp, ctypes.c_size_t, vp]
        L.bbc_search_host.argtypes = [vp, vp, i64, i32, i32, i64, vp, vp, vp, ctypes.c_size_t, vp]
        L.bbc_search_debug.argtypes = [vp, vp, i64, i32, i32, i64, vp, vp, vp, ctypes.c_size_t, vp,
                                       ctypes.POINTER(DebugBufs)]
        L.bbc_query_capacity.argtypes = [vp, i32, ctypes.POINTER(i64)]
        L.bbc_nccl_unique_id.argtypes = [vp]
        L.bbc_comm_init.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
        L.bbc_search_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int, vp, i64, i32, i32, i64, vp,
                                       vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t), vp]
        L.bbc_set_timing.argtypes = [vp, ctypes.c_int]
        L.bbc_set_probe_mode.argtypes = [vp, i32]
        L.bbc_set_scan_mode.argtypes = [vp, i32]
        L.bbc_set_buckets.argtypes = [vp, i32]
        L.bbc_set_rerank_order.argtypes = [vp, i32]
        L.bbc_set_remap.argtypes = [vp, i32]
        L.bbc_set_code_loads.argtypes = [vp, i32]
        L.bbc_set_scan_order.argtypes = [vp, i32]
        L.bbc_set_bound_rerank.argtypes = [vp, i32, ctypes.c_float]
        L.bbc_set_early_rerank.argtypes = [vp, i32]
        L.bbc_measure_smem_lookups.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_double)]
        L.bbc_measure_l2_read.argtypes = [i32, ctypes.c_size_t, i32, ctypes.POINTER(ctypes.c_double)]
        L.bbc_stats_vector.argtypes = [vp, ctypes.POINTER(i64), i32]
        L.bbc_get_timing.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int64)]
        L.bbc_last_stats.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(i64)]
        L.bbc_last_stats2.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                      ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.bbc_launch_count.argtypes = []
        L.bbc_launch_count.restype = i64
        L.bbc_last_error.argtypes = []
        L.bbc_last_error.restype = ctypes.c_char_p
        for fn in ("ivf_load", "bbc_index_info", "bbc_workspace_size", "bbc_search",
                   "bbc_search_host", "bbc_search_debug", "bbc_set_timing", "bbc_get_timing",
                   "bbc_last_stats", "bbc_query_capacity", "bbc_nccl_unique_id",
                   "bbc_comm_init", "bbc_search_group", "bbc_last_stats2", "bbc_set_probe_mode",
                   "bbc_set_scan_mode", "bbc_stats_vector", "bbc_set_buckets",
                   "bbc_set_rerank_order", "bbc_measure_l2_read", "bbc_set_remap",
                   "bbc_set_code_loads", "bbc_measure_smem_lookups", "bbc_set_scan_order", "bbc_set_bound_rerank",
                   "bbc_set_early_rerank"):
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise BBCError(f"bbc status {status}: {lib().bbc_last_error().decode()}")


def launch_count() -> int:
    return int(lib().bbc_launch_count())


def measure_l2_read_gbs(device: int = 0, nbytes: int = 48 << 20, reps: int = 20) -> float:
    """L2 -> SM read bandwidth (GB/s) of `device` (bbc_measure_l2_read; the roofline of the
    list-order re-rank)."""
    v = ctypes.c_double()
    _check(lib().bbc_measure_l2_read(int(device), int(nbytes), int(reps), ctypes.byref(v)))
    return v.value


def measure_smem_lookups(device: int = 0, rounds: int = 4096) -> float:
    """Shared-memory lookup rate (G lookups/s) of `device`: conflict-free 4-byte reads, one
    wavefront per warp instruction (bbc_measure_smem_lookups; the roofline of the PQ scan's LUT
    lookups)."""
    v = ctypes.c_double()
    _check(lib().bbc_measure_smem_lookups(int(device), int(rounds), ctypes.byref(v)))
    return v.value


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise BBCError("no CUDA device: the BBC path has no CPU fallback")
    return torch


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().bbc_nccl_unique_id(buf))
    return buf.raw


def _check_queries(q, d: int, device: int) -> None:
    """The C ABI takes no d: a query matrix of the wrong shape or device would be read past its
    end, so the binding checks it (2-D, d columns, fp32, contiguous, on the index's device)."""
    torch = _torch()
    if not (isinstance(q, torch.Tensor) and q.is_cuda and q.dtype == torch.float32
            and q.is_contiguous() and q.ndim == 2 and q.shape[1] == d and q.device.index == device):
        raise BBCError(f"queries must be a contiguous cuda:{device} float32 tensor [nq, {d}]")


def _check_out(out, nq: int, k: int, device=None) -> None:
    """Caller-supplied outputs: (ids int64 [nq, k], d2 float32 [nq, k]), contiguous, on the device
    (device None: host numpy arrays)."""
    ids, d2 = out
    if device is None:
        ok = (isinstance(ids, np.ndarray) and isinstance(d2, np.ndarray) and ids.dtype == np.int64
              and d2.dtype == np.float32 and ids.shape == (nq, k) and d2.shape == (nq, k)
              and ids.flags.c_contiguous and d2.flags.c_contiguous)
    else:
        torch = _torch()
        ok = (ids.dtype == torch.int64 and d2.dtype == torch.float32
              and tuple(ids.shape) == (nq, k) and tuple(d2.shape) == (nq, k)
              and ids.is_contiguous() and d2.is_contiguous() and ids.is_cuda and d2.is_cuda
              and ids.device.index == device and d2.device.index == device)
    if not ok:
        raise BBCError(f"out must be (int64 [{nq}, {k}], float32 [{nq}, {k}]) contiguous "
                       + ("host arrays" if device is None else f"cuda:{device} tensors"))


def search_group(shards, q, k: int, nprobe: int, budget: int, out=None, stream=None):
    """Sharded search over shards (Index objects loaded with rank i, world len(shards)) held by
    this process on one device: exchange steps are device reductions (bbc_search_group)."""
    torch = _torch()
    nq = q.shape[0]
    G = len(shards)
    for s in shards:
        _check_queries(q, s.info.d, s.device)
    if out is None:
        out = (torch.empty((nq, k), dtype=torch.int64, device=q.device),
               torch.empty((nq, k), dtype=torch.float32, device=q.device))
    _check_out(out, nq, k, shards[0].device)
    wss = [s.workspace(nq, k, nprobe, budget) for s in shards]
    hs = (ctypes.c_void_p * G)(*[s._h.value for s in shards])
    wp = (ctypes.c_void_p * G)(*[w.data_ptr() for w in wss])
    wb = (ctypes.c_size_t * G)(*[w.numel() for w in wss])
    st = torch.cuda.current_stream(q.device).cuda_stream if stream is None else stream
    _check(lib().bbc_search_group(hs, G, q.data_ptr(), nq, k, nprobe, budget, out[0].data_ptr(),
                                  out[1].data_ptr(), wp, wb, st))
    return out


class Index:
    """A loaded (shard of an) IVF index on one GPU (ivf_load / ivf_free)."""

    def __init__(self, path: str, rank: int = 0, world: int = 1, device: int | None = None):
        torch = _torch()
        dev = torch.cuda.current_device() if device is None else device
        self.device = dev
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().ivf_load(path.encode(), rank, world, dev, ctypes.byref(h)))
        self._h = h
        info = IndexInfo()
        _check(lib().bbc_index_info(h, ctypes.byref(info)))
        self.info = info
        self._ws = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ivf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ workspace
    def workspace_size(self, nq: int, k: int, nprobe: int, budget: int):
        b, m = ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().bbc_workspace_size(self._h, nq, k, nprobe, budget, ctypes.byref(b),
                                        ctypes.byref(m)))
        return b.value, m.value

    def workspace(self, nq: int, k: int, nprobe: int, budget: int, max_bytes: int | None = None):
        """A cached device workspace (uint8 tensor) big enough for nq queries in one micro-batch,
        capped at max_bytes (default 40% of the device memory; the library then processes the
        queries in micro-batches), never below the minimum."""
        torch = _torch()
        want, mn = self.workspace_size(nq, k, nprobe, budget)
        if max_bytes is None:          # default: at most 40% of the device; queries micro-batch
            max_bytes = int(0.4 * torch.cuda.get_device_properties(self.device).total_memory)
        want = max(mn, min(want, max_bytes))
        if self._ws is None or self._ws.numel() < want:
            self._ws = None
            self._ws = torch.empty(want, dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    # ------------------------------------------------------------------ search
    def search(self, q, k: int, nprobe: int, budget: int, out=None, workspace=None, stream=None):
        """q: cuda fp32 [nq, d] -> (ids int64 [nq, k], d2 fp32 [nq, k]) on the same device."""
        torch = _torch()
        _check_queries(q, self.info.d, self.device)
        nq = q.shape[0]
        if out is None:
            out = (torch.empty((nq, k), dtype=torch.int64, device=q.device),
                   torch.empty((nq, k), dtype=torch.float32, device=q.device))
        _check_out(out, nq, k, self.device)
        ws = self.workspace(nq, k, nprobe, budget) if workspace is None else workspace
        st = torch.cuda.current_stream(q.device).cuda_stream if stream is None else stream
        _check(lib().bbc_search(self._h, q.data_ptr(), nq, k, nprobe, budget, out[0].data_ptr(),
                                out[1].data_ptr(), ws.data_ptr(), ws.numel(), st))
        return out

    def search_host(self, q: np.ndarray, k: int, nprobe: int, budget: int, out=None,
                    workspace=None, stream=None):
        """Host arrays in and out (bbc_search_host); pinned numpy views are fastest."""
        torch = _torch()
        q = np.ascontiguousarray(q, dtype=np.float32)
        if q.ndim != 2 or q.shape[1] != self.info.d:
            raise BBCError(f"queries must be [nq, {self.info.d}]")
        nq = q.shape[0]
        if out is None:
            out = (np.empty((nq, k), dtype=np.int64), np.empty((nq, k), dtype=np.float32))
        _check_out(out, nq, k)
        ws = self.workspace(nq, k, nprobe, budget) if workspace is None else workspace
        st = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        _check(lib().bbc_search_host(self._h, q.ctypes.data, nq, k, nprobe, budget,
                                     out[0].ctypes.data, out[1].ctypes.data, ws.data_ptr(),
                                     ws.numel(), st))
        return out

    def search_debug(self, q, k: int, nprobe: int, budget: int, want_est: bool = False,
                     cand_stride: int | None = None):
        """Search plus every intermediate (parity tests).  Returns (ids, d2, dict of tensors).
        cand_stride: per-query capacity of the candidate buffers (default: the probed-object
        capacity; candidates past it are not copied, n_cand still counts them)."""
        torch = _torch()
        _check_queries(q, self.info.d, self.device)
        nq = q.shape[0]
        dev = q.device
        ws = self.workspace(nq, k, nprobe, budget, max_bytes=1 << 62)
        cap = int(self.cap(nprobe))
        cs = cap if cand_stride is None else int(cand_stride)
        t = dict(
            probe=torch.empty((nq, nprobe), dtype=torch.int32, device=dev),
            rq2=torch.empty((nq, nprobe), dtype=torch.float32, device=dev),
            nsample=torch.empty(nq, dtype=torch.int32, device=dev),
            edges=torch.empty((nq, 2), dtype=torch.float32, device=dev),
            hist=torch.empty((nq, 256), dtype=torch.int32, device=dev),
            tau=torch.empty(nq, dtype=torch.int32, device=dev),
            n_probed=torch.empty(nq, dtype=torch.int32, device=dev),
            n_cand=torch.empty(nq, dtype=torch.int32, device=dev),
            cand_ids=torch.full((nq, cs), -1, dtype=torch.int64, device=dev),
            cand_d2=torch.empty((nq, cs), dtype=torch.float32, device=dev),
            tau_pred=torch.empty(nq, dtype=torch.int32, device=dev),
            cand_early=torch.zeros((nq, cs), dtype=torch.uint8, device=dev),
        )
        if want_est:
            t["est"] = torch.empty((nq, cap), dtype=torch.float32, device=dev)
        db = DebugBufs(t["probe"].data_ptr(), t["rq2"].data_ptr(), t["nsample"].data_ptr(),
                       t["edges"].data_ptr(), t["hist"].data_ptr(), t["tau"].data_ptr(),
                       t["n_probed"].data_ptr(), t["est"].data_ptr() if want_est else None, cap,
                       t["n_cand"].data_ptr(), t["cand_ids"].data_ptr(), t["cand_d2"].data_ptr(),
                       cs, t["tau_pred"].data_ptr(), t["cand_early"].data_ptr())
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        d2 = torch.empty((nq, k), dtype=torch.float32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _check(lib().bbc_search_debug(self._h, q.data_ptr(), nq, k, nprobe, budget,
                                      ids.data_ptr(), d2.data_ptr(), ws.data_ptr(), ws.numel(),
                                      st, ctypes.byref(db)))
        return ids, d2, t

    def cap(self, nprobe: int) -> int:
        """Per-query element capacity (bbc_query_capacity)."""
        c = ctypes.c_int64()
        _check(lib().bbc_query_capacity(self._h, nprobe, ctypes.byref(c)))
        return c.value

    # ------------------------------------------------------------------ multi-GPU
    def comm_init(self, nccl_id: bytes, rank: int, world: int) -> None:
        """Attach an NCCL communicator (SPMD sharded search; see include/bbc.h)."""
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().bbc_comm_init(self._h, buf, rank, world))

    # ------------------------------------------------------------------ instrumentation
    PROBE_SIMT, PROBE_TENSOR, PROBE_AUTO = 0, 1, 2

    def set_probe_mode(self, mode: int) -> None:
        """Step a1 on the CUDA cores (canonical d^2 everywhere, PROBE_SIMT), as the tensor-core
        shortlist + canonical re-score (PROBE_TENSOR), or chosen per search (PROBE_AUTO, the
        default: tensor cores when nprobe <= nlist / 16).  Same probe lists in every mode."""
        _check(lib().bbc_set_probe_mode(self._h, int(mode)))

    def set_buckets(self, nbuckets: int) -> None:
        """B regular buckets of the result buffer (1..255, default 255; Eq. 6, Table 4)."""
        _check(lib().bbc_set_buckets(self._h, int(nbuckets)))

    SCAN_SIMT, SCAN_TENSOR = 0, 1

    def set_scan_mode(self, mode: int) -> None:
        """RaBitQ estimates with popcounts per (query, list) (SCAN_SIMT) or as list-major integer
        GEMMs on the tensor cores (SCAN_TENSOR, default); PQ indexes ignore it."""
        _check(lib().bbc_set_scan_mode(self._h, int(mode)))

    def set_remap(self, m: int) -> None:
        """m equal-depth buckets from the sample (the paper's n_ew -> m remap, reading R6); 0
        (default) keeps the equal-width cells as the buckets."""
        _check(lib().bbc_set_remap(self._h, int(m)))

    ALG3_OFF, ALG3_LIST, ALG3_QUERY = 0, 1, 2

    def set_bound_rerank(self, on: bool, eps0: float = 1.9, gathers: str = "list") -> None:
        """Algorithm 3 (the bound-aware RaBitQ re-rank) in place of Algorithm 1's
        superset re-rank: lb/ub buckets from the RaBitQ bound with eps0 (1.9 in the paper), the
        marginal-bucket loop, exact d^2 of B_exact.  gathers="list": every candidate's exact
        distance by the list-order re-rank, then the loop (faster); "query": only B_exact's rows,
        gathered per query as the loop reaches them.  Same results.  RaBitQ, single shard."""
        if gathers not in ("list", "query"):
            raise BBCError("gathers must be 'list' or 'query'")
        mode = (self.ALG3_LIST if gathers == "list" else self.ALG3_QUERY) if on else self.ALG3_OFF
        _check(lib().bbc_set_bound_rerank(self._h, mode, float(eps0)))

    def set_early_rerank(self, on: bool) -> None:
        """Algorithm 4 (early re-ranking of IVF+PQ): straight after the scan pass,
        before the threshold is known, every object in a bucket below the predicted threshold
        tau_pred gets its exact distance; the re-rank computes the remaining candidates.  Same results as Algorithm 1.  8-bit PQ,
        single shard, equal-width buckets."""
        _check(lib().bbc_set_early_rerank(self._h, int(bool(on))))

    CODES_AUTO, CODES_CACHED, CODES_STREAM = 0, 1, 2

    def set_code_loads(self, mode: int) -> None:
        """L1 policy of the 8-bit PQ scan's code loads: cached (CODES_CACHED), streamed past L1
        (CODES_STREAM) or chosen from the codes' size against the L2 size (CODES_AUTO, default).
        Same results in every mode."""
        _check(lib().bbc_set_code_loads(self._h, int(mode)))

    ORDER_AUTO, ORDER_PROBE, ORDER_SWEEP = 0, 1, 2

    def set_scan_order(self, order: int) -> None:
        """Visiting order of the 8-bit PQ scan: probe order (ORDER_PROBE), lists by ascending id
        with work items issued by their first list (ORDER_SWEEP: codes shared through L2), or
        chosen from the codes' size against the L2 size (ORDER_AUTO, default).  Same results."""
        _check(lib().bbc_set_scan_order(self._h, int(order)))

    RERANK_QUERY, RERANK_LIST, RERANK_AUTO, RERANK_TILE = 0, 1, 2, 3

    def set_rerank_order(self, order: int) -> None:
        """Exact re-rank work order: per query (RERANK_QUERY), per (list, query) segment in list
        order (RERANK_LIST: rows shared by the queries of a list come from L2), list order with
        each list's rows staged in shared memory tile by tile (RERANK_TILE, fp32 rows <= 512 B),
        or chosen from the data size and reuse (RERANK_AUTO, default)."""
        _check(lib().bbc_set_rerank_order(self._h, int(order)))

    def set_timing(self, on: bool) -> None:
        _check(lib().bbc_set_timing(self._h, int(on)))

    def get_timing(self):
        arr = (ctypes.c_float * 8)()
        calls = ctypes.c_int64()
        _check(lib().bbc_get_timing(self._h, arr, 8, ctypes.byref(calls)))
        return dict(zip(STAGES, [float(x) for x in arr])), calls.value

    def last_stats(self):
        a, b, c, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().bbc_last_stats2(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                     ctypes.byref(d)))
        v = (ctypes.c_int64 * 9)()
        _check(lib().bbc_stats_vector(self._h, v, 9))
        return dict(probed=a.value, candidates=b.value, microbatches=c.value, sampled=d.value,
                    shortlisted=v[3], rerank_list_batches=v[5], sample_pass=v[6],
                    early_objects=v[7], early_candidates=v[8])
