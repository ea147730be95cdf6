"""Deterministic IVF index construction (k-means lists, PQ codebooks/codes, RaBitQ rotation/codes).

Seeded-input layer.  The index is an *input* of the query hot path: BASELINE.json north_star
"the oracle builds the index deterministically from the seed (k-means coarse quantizer, PQ
codebooks or RaBitQ rotation and factors) and serializes it so both paths query the same index".
The serialized file (datagen/index_file.py) is the contract; the CPU oracle and the
CUDA path both read it and share nothing else.  None of the query-time arithmetic (probe
distances, LUTs, estimates, buckets, threshold, re-rank, select) lives here.

Paper passages followed
  * IVF: "partitions the data vectors into n_cluster clusters using the k-means algorithm during
    indexing" (section 2 "Quantization").
  * PQ: "construct a quantization codebook, assign each data vector to their nearest codebook
    vector, and store the codebook ids as compact quantization codes".
    8-bit codes, M from BASELINE.json; raw (non-residual) encoding (reading R8).
  * RaBitQ (PAPER.md L106, L413, L1440 cite gao2024rabitq): random orthogonal rotation P,
    1 bit per rotated dimension of the normalised residual o = (o_r - c_L)/||o_r - c_L||,
    per-vector factors r_o = ||o_r - c_L|| and g_o = <o_bar, o> = sum_i |y_i| / sqrt(D) with
    y = P^T o.  D = d rounded up to a multiple of 64.

Determinism: every random choice comes from the config seed's `kmeans` / `quantizer` streams;
ties in assignments go to the smaller index (argmin semantics).  Assignments (k-means and PQ
encoding) use GEMM-form fp32 distances, so a near-tie may pick a codeword whose exact distance
exceeds the minimum by a rounding error; tests/test_datagen.py bounds that slack.  Heavy linear algebra runs
through torch (plumbing only) in chunks: on a CUDA device when one is present (cuBLAS fp32
GEMMs; BBC_BUILD_DEVICE=cpu forces the CPU), so an index built on a GPU box can differ from one
built on a CPU at near-ties -- the serialized file, not the build, is what both query paths share.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np
import torch

from . import synth
from .configs import Config

_CHUNK_ELEMS = 1 << 25   # elements of one distance tile (rows x centroids)


def _device() -> str:
    want = os.environ.get("BBC_BUILD_DEVICE", "auto")
    return "cuda" if want != "cpu" and torch.cuda.is_available() else "cpu"


def _assign(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Nearest centroid per row (GEMM-form fp32 distances; ties -> smaller id)."""
    dev = _device()
    Ct = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float32)).to(dev)
    cn = (Ct * Ct).sum(1)
    out = np.empty(len(X), dtype=np.int64)
    rows = max(1, _CHUNK_ELEMS // max(1, len(C)))
    with _NoTF32():
        for lo in range(0, len(X), rows):
            xb = torch.from_numpy(np.ascontiguousarray(X[lo:lo + rows], dtype=np.float32)).to(dev)
            dist = cn[None, :] - 2.0 * (xb @ Ct.T)
            out[lo:lo + len(xb)] = torch.argmin(dist, dim=1).cpu().numpy()
    return out


class _NoTF32:
    """fp32 GEMMs (no TF32 rounding of the inputs) while building."""

    def __enter__(self):
        self.prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False

    def __exit__(self, *a):
        torch.backends.cuda.matmul.allow_tf32 = self.prev


def kmeans(X: np.ndarray, K: int, iters: int, g: np.random.Generator, train_n: int) -> np.ndarray:
    """Lloyd's k-means.  Returns fp32 centroids [K x d].

    init = K distinct training points drawn with the seed; centroid sums in fp64; an empty
    cluster is re-seeded with a seeded member of the currently largest cluster.
    """
    N = len(X)
    tr = np.sort(g.choice(N, size=min(N, train_n), replace=False)) if train_n < N else np.arange(N)
    T = np.ascontiguousarray(X[tr], dtype=np.float32)
    C = T[np.sort(g.choice(len(T), size=K, replace=False))].astype(np.float64)
    for _ in range(iters):
        lab = _assign(T, C.astype(np.float32))
        cnt = np.bincount(lab, minlength=K)
        sums = np.zeros((K, T.shape[1]), dtype=np.float64)
        np.add.at(sums, lab, T.astype(np.float64)) if len(T) < 200_000 else _chunked_sum(sums, lab, T)
        nz = cnt > 0
        C[nz] = sums[nz] / cnt[nz, None]
        for e in np.flatnonzero(~nz):
            big = int(np.argmax(cnt))
            members = np.flatnonzero(lab == big)
            pick = members[g.integers(0, len(members))]
            C[e] = T[pick].astype(np.float64) + 1e-4 * g.standard_normal(T.shape[1])
            cnt[big] -= 1
            lab[pick] = e
            cnt[e] = 1
    return C.astype(np.float32)


def _chunked_sum(sums: np.ndarray, lab: np.ndarray, T: np.ndarray) -> None:
    order = np.argsort(lab, kind="stable")
    ls = lab[order]
    starts = np.flatnonzero(np.r_[True, ls[1:] != ls[:-1]])
    for lo in range(0, len(starts), 4096):
        s = starts[lo:lo + 4096]
        end = starts[lo + 4096] if lo + 4096 < len(starts) else len(order)
        blk = T[order[s[0]:end]].astype(np.float64)
        red = np.add.reduceat(blk, s - s[0], axis=0)
        sums[ls[s]] += red


def build(cfg: Config, X: np.ndarray | None = None, verbose: bool = False) -> dict:
    """Build the IVF index of `cfg` from its seed.  Returns the dict `index_file.write` takes."""
    if X is None:
        X = synth.generate_data(cfg)
    st = synth.streams(cfg.seed)
    gk = synth.rng(st["kmeans"])
    gq = synth.rng(st["quantizer"])
    N, d = X.shape
    Xf = X if X.dtype == np.float32 else None

    def rows_f32(lo, hi):
        return X[lo:hi] if Xf is not None else X[lo:hi].astype(np.float32)

    train_n = cfg.kmeans_train_per_list * cfg.nlist
    cent = kmeans(X, cfg.nlist, cfg.kmeans_iters, gk, train_n)
    lab = np.empty(N, dtype=np.int64)
    for lo in range(0, N, 1 << 20):
        lab[lo:lo + (1 << 20)] = _assign(rows_f32(lo, min(N, lo + (1 << 20))), cent)
    order = np.argsort(lab, kind="stable")                 # lists ordered by (list id, point id)
    sizes = np.bincount(lab, minlength=cfg.nlist)
    offsets = np.zeros(cfg.nlist + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    if cfg.metric == "ip" and cfg.kind != "pq":
        raise ValueError("the inner-product metric is built for PQ indexes only")
    out = dict(kind=cfg.kind, raw_dtype=cfg.raw_dtype, N=N, d=d, nlist=cfg.nlist, seed=cfg.seed,
               metric=cfg.metric,
               centroids=cent, list_offsets=offsets, ids=order.astype(np.int64),
               raw=np.ascontiguousarray(X[order]))
    if verbose:
        print(f"[build] {cfg.name}: lists built, sizes min {sizes.min()} max {sizes.max()}", file=sys.stderr)
    if cfg.kind == "pq":
        M, ds = cfg.M, cfg.dsub
        trq = np.sort(gq.choice(N, size=min(N, cfg.pq_train), replace=False))
        Tq = X[trq].astype(np.float32)
        ksub = 1 << cfg.pq_bits
        books = np.empty((M, ksub, ds), dtype=np.float32)
        for m in range(M):
            books[m] = kmeans(Tq[:, m * ds:(m + 1) * ds], ksub, cfg.pq_iters, gq, len(Tq))
        codes = np.empty((N, M), dtype=np.uint8)
        raw = out["raw"]
        for lo in range(0, N, 1 << 18):
            blk = raw[lo:lo + (1 << 18)].astype(np.float32)
            for m in range(M):
                codes[lo:lo + len(blk), m] = _assign(blk[:, m * ds:(m + 1) * ds], books[m])
        out.update(M=M, nbits=cfg.pq_bits, codebooks=books, codes=codes)
    else:
        D = ((d + 63) // 64) * 64
        G = gq.standard_normal((D, D))
        Qm, R = np.linalg.qr(G)
        Qm = Qm * np.sign(np.diag(R))[None, :]
        P = Qm.astype(np.float32)
        P64 = P.astype(np.float64)
        cpad = np.zeros((cfg.nlist, D), dtype=np.float64)
        cpad[:, :d] = cent
        wL = (cpad @ P64).astype(np.float32)                # w_L = P^T c_L
        bits = np.zeros((N, D // 8), dtype=np.uint8)
        fac = np.zeros((N, 2), dtype=np.float32)
        raw = out["raw"]
        ll = np.repeat(np.arange(cfg.nlist), sizes)
        for lo in range(0, N, 1 << 16):
            hi = min(N, lo + (1 << 16))
            diff = np.zeros((hi - lo, D), dtype=np.float64)
            diff[:, :d] = raw[lo:hi].astype(np.float64) - cent[ll[lo:hi]].astype(np.float64)
            r = np.sqrt((diff * diff).sum(1))
            zero = r == 0
            o = diff / np.where(zero, 1.0, r)[:, None]
            y = o @ P64                                      # y = P^T o
            b = y >= 0
            b[zero] = True
            gO = np.abs(y).sum(1) / math.sqrt(D)
            gO[zero] = 1.0
            bits[lo:hi] = np.packbits(b, axis=1, bitorder="little")
            fac[lo:hi, 0] = r
            fac[lo:hi, 1] = gO
        out.update(M=0, nbits=1, D=D, P=P, wL=wL, bits=bits, factors=fac)
    return out
