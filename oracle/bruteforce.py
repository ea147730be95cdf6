"""Exact ground truth and accuracy metrics -- TEST INFRASTRUCTURE ONLY (see bbc_oracle.py header).

  * brute-force top-k ("ground-truth result computed by the brute-force search", PAPER.md
    L1433): fp64 squared L2 over the whole database, ties broken by id.
  * recall@k = |R ∩ R~| / k, tie-tolerant: a returned id also counts when its
    exact distance is <= the k-th ground-truth distance (reading R14).
  * relative error: mean over ranks of Dist(q, R[i]) / Dist(q, R~[i]) - 1, both
    lists sorted ascending, over ranks 1..k (reading R15), Dist = Euclidean (not squared).
"""
from __future__ import annotations

import numpy as np


def exact_all(q: np.ndarray, X: np.ndarray, chunk: int = 1 << 18, metric: str = "l2") -> np.ndarray:
    """fp64 ||q - x||^2 for every row of X (norm expansion in fp64); inner product: -<q, x>."""
    q64 = np.asarray(q, dtype=np.float64)
    qn = q64 @ q64
    out = np.empty(len(X), dtype=np.float64)
    for lo in range(0, len(X), chunk):
        xb = np.asarray(X[lo:lo + chunk], dtype=np.float64)
        if metric == "ip":
            out[lo:lo + len(xb)] = -(xb @ q64)
        else:
            out[lo:lo + len(xb)] = np.maximum(0.0, qn + (xb * xb).sum(1) - 2.0 * (xb @ q64))
    return out


def ground_truth(Q: np.ndarray, X: np.ndarray, k: int, metric: str = "l2"):
    """(ids int64 [nq x k], d2 fp64 [nq x k]) of the exact k nearest rows (smallest keys),
    ordered by (key, id)."""
    nq = len(Q)
    gi = np.empty((nq, k), dtype=np.int64)
    gd = np.empty((nq, k), dtype=np.float64)
    ids = np.arange(len(X))
    for i in range(nq):
        d2 = exact_all(Q[i], X, metric=metric)
        cand = np.argpartition(d2, k - 1)[:k] if k < len(X) else ids
        kth = d2[cand].max()
        cand = np.flatnonzero(d2 <= kth)                  # keep every tie of the k-th distance
        order = cand[np.lexsort((cand, d2[cand]))][:k]
        gi[i] = order
        gd[i] = d2[order]
    return gi, gd


def recall(res_ids: np.ndarray, res_d2_exact64: np.ndarray, gt_ids: np.ndarray,
           gt_d2: np.ndarray) -> float:
    """Mean tie-tolerant recall@k over queries.  res_d2_exact64: fp64 exact d^2 of res_ids."""
    nq, k = gt_ids.shape
    tot = 0
    for i in range(nq):
        ok = res_ids[i] >= 0
        inset = np.isin(res_ids[i], gt_ids[i])
        tie = res_d2_exact64[i] <= gt_d2[i, -1]
        tot += int(np.count_nonzero(ok & (inset | tie)))
    return tot / (nq * k)


def relative_error(res_d2: np.ndarray, gt_d2: np.ndarray) -> float:
    r = np.sqrt(np.sort(np.asarray(res_d2, dtype=np.float64), axis=1))
    g = np.sqrt(np.sort(np.asarray(gt_d2, dtype=np.float64), axis=1))
    m = g > 0
    return float(np.mean(r[m] / g[m] - 1.0))
