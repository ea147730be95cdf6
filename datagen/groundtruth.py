"""Ground truth and accuracy metrics of a workload (measurement side of the seeded-input layer).

Used by bench.py to report recall@k of the GPU results; it is not part of the query path and
holds none of its arithmetic.  Definitions (section 4.1):
  * ground truth = brute-force exact top-k (fp64 squared L2, ties by id);
  * recall@k = |R ∩ R~| / k, tie-tolerant (an id also counts when its exact distance is <= the
    k-th ground-truth distance; reading R14);
  * relative error = mean over ranks 1..k of Dist(R[i]) / Dist(R~[i]) - 1 (Euclidean, sorted).
"""
from __future__ import annotations

import os

import numpy as np


def _sqdist(Q: np.ndarray, X: np.ndarray, chunk: int = 1 << 17, metric: str = "l2") -> np.ndarray:
    """fp64 keys: squared L2, or -<q, x> for the inner-product metric."""
    Q64 = np.asarray(Q, dtype=np.float64)
    qn = (Q64 * Q64).sum(1)
    out = np.empty((len(Q), len(X)), dtype=np.float64)
    for lo in range(0, len(X), chunk):
        xb = np.asarray(X[lo:lo + chunk], dtype=np.float64)
        if metric == "ip":
            out[:, lo:lo + len(xb)] = -(Q64 @ xb.T)
        else:
            out[:, lo:lo + len(xb)] = np.maximum(0.0, qn[:, None] + (xb * xb).sum(1)[None] - 2.0 * (Q64 @ xb.T))
    return out


def topk(Q: np.ndarray, X: np.ndarray, k: int, block: int = 16, metric: str = "l2"):
    """(ids int64 [nq x k], d2 fp64 [nq x k]) exact, ordered by (d2, id)."""
    nq = len(Q)
    gi = np.empty((nq, k), dtype=np.int64)
    gd = np.empty((nq, k), dtype=np.float64)
    for lo in range(0, nq, block):
        D = _sqdist(Q[lo:lo + block], X, metric=metric)
        for r in range(len(D)):
            d = D[r]
            cand = np.argpartition(d, k - 1)[:k] if k < len(d) else np.arange(len(d))
            kth = d[cand].max()
            cand = np.flatnonzero(d <= kth)
            order = cand[np.lexsort((cand, d[cand]))][:k]
            gi[lo + r] = order
            gd[lo + r] = d[order]
    return gi, gd


def topk_cuda(Q: np.ndarray, X: np.ndarray, k: int, metric: str = "l2", block: int = 8):
    """Same as topk (fp64 keys by the same norm expansion, ties of the k-th key kept and ordered
    by (key, id)) with the fp64 arithmetic on a CUDA device through torch: measurement plumbing,
    not the query path.  X is streamed to the device once in row chunks per query block."""
    import torch
    dev = torch.device("cuda")
    nq, N = len(Q), len(X)
    gi = np.empty((nq, k), dtype=np.int64)
    gd = np.empty((nq, k), dtype=np.float64)
    chunk = 1 << 21
    Xd = [torch.from_numpy(np.ascontiguousarray(X[lo:lo + chunk])).to(dev) for lo in range(0, N, chunk)]
    xn = [(x.double() * x.double()).sum(1) for x in Xd] if metric != "ip" else None
    for lo in range(0, nq, block):
        qb = torch.from_numpy(np.asarray(Q[lo:lo + block], dtype=np.float64)).to(dev)
        qn = (qb * qb).sum(1)
        D = torch.empty((len(qb), N), dtype=torch.float64, device=dev)
        c0 = 0
        for j, x in enumerate(Xd):
            xb = x.double()
            if metric == "ip":
                D[:, c0:c0 + len(xb)] = -(qb @ xb.T)
            else:
                D[:, c0:c0 + len(xb)] = torch.clamp(qn[:, None] + xn[j][None, :] - 2.0 * (qb @ xb.T), min=0.0)
            c0 += len(xb)
        kth = torch.topk(D, k, dim=1, largest=False).values.max(dim=1).values
        for r in range(len(qb)):
            cand = torch.nonzero(D[r] <= kth[r]).squeeze(1).cpu().numpy()
            d = D[r, torch.from_numpy(cand).to(dev)].cpu().numpy()
            order = np.lexsort((cand, d))[:k]
            gi[lo + r] = cand[order]
            gd[lo + r] = d[order]
        del D
    return gi, gd


def cached_topk(tag: str, Q: np.ndarray, X: np.ndarray, k: int, cache_dir: str, metric: str = "l2"):
    path = os.path.join(cache_dir, f"gt_{tag}_{len(Q)}_{k}.npz")
    if os.path.exists(path):
        z = np.load(path)
        return z["ids"], z["d2"]
    try:
        import torch
        cuda = torch.cuda.is_available()
    except Exception:
        cuda = False
    gi, gd = topk_cuda(Q, X, k, metric=metric) if cuda else topk(Q, X, k, metric=metric)
    np.savez(path, ids=gi, d2=gd)
    return gi, gd


def exact_of(Q: np.ndarray, X: np.ndarray, ids: np.ndarray, metric: str = "l2") -> np.ndarray:
    """fp64 exact keys of the returned ids (inf for padding ids < 0)."""
    out = np.full(ids.shape, np.inf)
    for i in range(len(Q)):
        ok = ids[i] >= 0
        rows = np.asarray(X[ids[i][ok]], dtype=np.float64)
        if metric == "ip":
            out[i][ok] = -(rows @ Q[i].astype(np.float64))
        else:
            out[i][ok] = ((rows - Q[i].astype(np.float64)) ** 2).sum(1)
    return out


def recall(ids: np.ndarray, d2_exact: np.ndarray, gt_ids: np.ndarray, gt_d2: np.ndarray) -> float:
    nq, k = gt_ids.shape
    hit = 0
    for i in range(nq):
        ok = ids[i] >= 0
        hit += int(np.count_nonzero(ok & (np.isin(ids[i], gt_ids[i]) | (d2_exact[i] <= gt_d2[i, -1]))))
    return hit / (nq * k)


def relative_error(d2: np.ndarray, gt_d2: np.ndarray) -> float:
    """Squared-L2 keys only (Euclidean ratios); None-free: callers skip it for inner product."""
    r = np.sqrt(np.sort(np.asarray(d2, dtype=np.float64), axis=1))
    g = np.sqrt(np.sort(np.asarray(gt_d2, dtype=np.float64), axis=1))
    m = (g > 0) & np.isfinite(r)
    return float(np.mean(r[m] / g[m] - 1.0))
