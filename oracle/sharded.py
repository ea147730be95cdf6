"""Oracle of the list-sharded query path -- TEST INFRASTRUCTURE ONLY (see bbc_oracle.py header).

Each rank holds the IVF lists assigned to it and talks to the others only through `allreduce`
(sum or min of an integer/float numpy array, e.g. torch.distributed over gloo).  The exchange
steps are the ones DESIGN.md section 6 specifies for the GPU path:

  * shard assignment: lists by (size desc, id asc), each to the currently least-loaded rank
    (ties to the lowest rank);
  * d_min = MIN over ranks of the local sample minimum; d_max = budget-th smallest sample
    estimate over all ranks, found digit by digit (4 x 8 bits of the ordered fp32 key) from
    all-reduced 256-bin histograms;
  * the bucket histogram is all-reduced (sum), so every rank applies one threshold bucket;
  * the k smallest (exact d^2, id) keys over all ranks: 8 x 8-bit digits of the 64-bit key from
    all-reduced 256-bin histograms; the per-(rank, query) counts of selected pairs are all-reduced,
    and every rank's selected (d^2, id) pairs, packed query after query, are all-gathered
    (north_star: "an all-gather of (distance, id) pairs feeds the final top-k"); each rank places
    rank r's pairs of query q after those of ranks < r, so every rank holds the whole result.

It reuses the per-rank arithmetic of bbc_oracle (probe, LUT, estimates, buckets, exact d^2) and
must reproduce bbc_oracle.search exactly (tests/test_sharded_gloo.py).
"""
from __future__ import annotations

import numpy as np

from . import bbc_oracle as O


def assign_lists(sizes: np.ndarray, world: int) -> np.ndarray:
    """owner[L] for every list (greedy balance, as ivf_load does)."""
    order = sorted(range(len(sizes)), key=lambda L: (-int(sizes[L]), L))
    load = [0] * world
    owner = np.zeros(len(sizes), dtype=np.int64)
    for L in order:
        r = min(range(world), key=lambda i: (load[i], i))
        owner[L] = r
        load[r] += int(sizes[L])
    return owner


def f2key(x: np.ndarray) -> np.ndarray:
    """Monotone map fp32 -> uint32 (same total order as the float values)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & 0x80000000) != 0
    return np.where(neg, (~u) & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)


def key2f(k: int) -> np.float32:
    k = int(k)
    u = (k & 0x7FFFFFFF) if (k & 0x80000000) else ((~k) & 0xFFFFFFFF)
    return np.array([u], dtype=np.uint32).view(np.float32)[0]


def radix_select(local_keys: np.ndarray, need: int, nbits: int, allreduce) -> int:
    """The need-th smallest key (1-based) of the union over ranks, 8 bits at a time."""
    prefix = 0
    for shift in range(nbits - 8, -1, -8):
        if shift + 8 >= 64:
            m = np.ones(len(local_keys), bool)
        else:
            m = (local_keys >> np.uint64(shift + 8)) == np.uint64(prefix >> (shift + 8))
        digits = ((local_keys[m] >> np.uint64(shift)) & np.uint64(255)).astype(np.int64)
        h = allreduce(np.bincount(digits, minlength=256).astype(np.int64), "sum")
        c = np.cumsum(h)
        dgt = int(np.searchsorted(c, need, side="left"))
        need -= int(c[dgt - 1]) if dgt > 0 else 0
        prefix |= dgt << shift
    return prefix


def search(ix: dict, Q: np.ndarray, k: int, nprobe: int, budget: int, rank: int, world: int,
           allreduce, allgather):
    """allreduce(array, "sum" | "min") -> array; allgather(array) -> list of every rank's array
    (rank order, sizes may differ)."""
    off = np.asarray(ix["list_offsets"])
    gsize = np.diff(off)
    owner = assign_lists(gsize, world)
    pr, rq = O.probe(np.asarray(Q, dtype=np.float32), ix["centroids"], nprobe)
    nq = len(Q)
    mine_sel = []                                         # per query: this rank's selected pairs
    for i in range(nq):
        lists = pr[i]
        s = O.sample_lists(gsize[lists], budget)          # global sizes: same on every rank
        mine = [j for j in range(nprobe) if owner[lists[j]] == rank]
        est_parts, pos_parts, samp = [], [], []
        if ix["kind"] == "pq":
            lut = O.pq_lut(Q[i], ix["codebooks"])
        else:
            u = O.rabitq_rotate(Q[i], ix["P"])
        for j in mine:
            L = lists[j]
            sl = slice(off[L], off[L + 1])
            if ix["kind"] == "pq":
                e = O.pq_est(lut, np.asarray(ix["codes"][sl]))
            else:
                qbar, cs, r = O.rabitq_query_code(u, ix["wL"][L], rq[i, j])
                e = O.rabitq_est(np.asarray(ix["bits"][sl]), np.asarray(ix["factors"][sl]), qbar,
                                 cs, r, rq[i, j])
            est_parts.append(e)
            pos_parts.append(np.arange(off[L], off[L + 1]))
            samp.append(np.full(len(e), j < s))
        est = np.concatenate(est_parts) if est_parts else np.zeros(0, np.float32)
        pos = np.concatenate(pos_parts) if pos_parts else np.zeros(0, np.int64)
        insamp = np.concatenate(samp) if samp else np.zeros(0, bool)
        if s == 0:
            keep = np.ones(len(est), bool)
        else:
            skeys = f2key(est[insamp])
            kmin = allreduce(np.array([skeys.min() if len(skeys) else 0xFFFFFFFF], np.int64), "min")[0]
            kmax = radix_select(skeys, budget, 32, allreduce)
            dmin, dmax = key2f(kmin), key2f(kmax)
            cell = O.cells(est, dmin, dmax)
            H = allreduce(np.bincount(cell, minlength=256).astype(np.int64), "sum")
            tau = O.threshold(H, budget)
            keep = cell <= tau
        spos = pos[keep]
        sid = np.asarray(ix["ids"][spos])
        d2 = O.exact_d2(Q[i], np.asarray(ix["raw"][spos]))
        total = int(allreduce(np.array([len(sid)], np.int64), "sum")[0])
        keys = (f2key(d2) << np.uint64(32)) | sid.astype(np.uint64)
        if total > k:
            thr = radix_select(keys, k, 64, allreduce)
            chosen = keys <= np.uint64(thr)
        else:
            chosen = np.ones(len(keys), bool)
        order = np.flatnonzero(chosen)                    # candidate (probe) order
        mine_sel.append((sid[order], d2[order]))
    # counts of selected pairs per (rank, query), all-reduced: every rank knows every offset
    cnt = np.zeros((world, nq), np.int64)
    cnt[rank] = [len(x[0]) for x in mine_sel]
    cnt = allreduce(cnt, "sum")
    # this rank's pairs packed query after query, as (fp32 bits of d^2) << 32 | id
    packed = np.concatenate(
        [(np.asarray(d, np.float32).view(np.uint32).astype(np.uint64) << np.uint64(32))
         | np.asarray(i_, np.uint64) for i_, d in mine_sel]) if nq else np.zeros(0, np.uint64)
    parts = allgather(packed)
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_d2 = np.full((nq, k), np.inf, dtype=np.float32)
    fill = np.zeros(nq, np.int64)
    for r in range(world):                                # rank r's pairs after those of ranks < r
        pr_ = np.asarray(parts[r], np.uint64)
        assert len(pr_) == int(cnt[r].sum())
        o = 0
        for i in range(nq):
            c = int(cnt[r, i])
            blk = pr_[o:o + c]
            out_ids[i, fill[i]:fill[i] + c] = (blk & np.uint64(0xFFFFFFFF)).astype(np.int64)
            out_d2[i, fill[i]:fill[i] + c] = (blk >> np.uint64(32)).astype(np.uint32).view(np.float32)
            fill[i] += c
            o += c
    return out_ids, out_d2
