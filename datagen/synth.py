"""Seeded synthetic workloads shaped like the paper's datasets (stand-ins).

Part of the seeded-input layer: random numbers only, no part of the BBC query arithmetic.

The paper evaluates on Wiki, C4, MSMARCO and Deep100M (Table 1), none of
which is available here.  BASELINE.json configs[0..4] name synthetic distributions instead; the
underspecified parts are filled in as SURVEY.md section 8(d) proposes:

  C1  256 centres mu_j ~ N(0, I_128); x = mu_j + 0.3 z; uniform component weights.   (fp32)
  C2  1,024 prototypes; per (prototype, dim) scale g ~ Gamma(2, 0.5);
      x_t = min(255, floor(Exp(mean 20 g))); dims 64..127 zeroed with prob. 0.7.   (integer fp32)
  C3  x = 0.5 u + 0.5 (0.5 + 0.2887 z W), u ~ U[0,1]^960, z ~ N(0, I_64),
      W_ij ~ N(0, 1/64) fixed per seed (rank-64 correlated component).           (fp32)
  C4  c_j = normalize(N(0, I_96)), 1,024 components; x = normalize(c_j + 0.06 z).   (fp32, unit norm)
  C5  mu_{j,t} = min(255, floor(Exp(mean 32))), 4,096 components;
      x = clip(round(mu_j + 8 z), 0, 255).                                        (uint8)

Streams: numpy Generator(PCG64) over SeedSequence(seed).spawn(): {structure, data, queries,
kmeans, quantizer}.  Data rows are generated in 1M-row chunks, each from its own spawned child of
the data stream, so any chunk can be regenerated independently.  Queries are fresh held-out draws
(SURVEY 8(c) ambiguity #16) in 256-query blocks, so the first n queries do not depend on nq.
"""
from __future__ import annotations

import numpy as np

from .configs import Config

CHUNK = 1_000_000
_STREAMS = ("structure", "data", "queries", "kmeans", "quantizer")


def streams(seed: int) -> dict:
    ss = np.random.SeedSequence(seed)
    return dict(zip(_STREAMS, ss.spawn(len(_STREAMS))))


def rng(seq: np.random.SeedSequence) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seq))


def _structure(cfg: Config, st: dict) -> dict:
    g = rng(st["structure"])
    d = cfg.d
    if cfg.gen == "C1":
        return {"mu": g.standard_normal((256, d))}
    if cfg.gen == "C2":
        scale = g.gamma(2.0, 0.5, size=(1024, d))
        return {"scale": scale}
    if cfg.gen == "C3":
        return {"W": g.standard_normal((64, d)) / 8.0}
    if cfg.gen == "C4":
        c = g.standard_normal((1024, d))
        c /= np.linalg.norm(c, axis=1, keepdims=True)
        return {"c": c}
    if cfg.gen == "C5":
        mu = np.minimum(255.0, np.floor(g.exponential(32.0, size=(4096, d))))
        return {"mu": mu}
    raise ValueError(cfg.gen)


def _draw(cfg: Config, S: dict, g: np.random.Generator, n: int) -> np.ndarray:
    d = cfg.d
    if cfg.gen == "C1":
        comp = g.integers(0, 256, size=n)
        x = S["mu"][comp] + 0.3 * g.standard_normal((n, d))
        return x.astype(np.float32)
    if cfg.gen == "C2":
        comp = g.integers(0, 1024, size=n)
        x = np.floor(g.exponential(1.0, size=(n, d)) * (20.0 * S["scale"][comp]))
        np.minimum(x, 255.0, out=x)
        half = d // 2
        zero = g.random((n, d - half)) < 0.7
        x[:, half:][zero] = 0.0
        return x.astype(np.float32)
    if cfg.gen == "C3":
        u = g.random((n, d))
        z = g.standard_normal((n, 64))
        x = 0.5 * u + 0.5 * (0.5 + 0.2887 * (z @ S["W"]))
        return x.astype(np.float32)
    if cfg.gen == "C4":
        comp = g.integers(0, 1024, size=n)
        x = S["c"][comp] + 0.06 * g.standard_normal((n, d))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        return x.astype(np.float32)
    if cfg.gen == "C5":
        comp = g.integers(0, 4096, size=n)
        x = np.rint(S["mu"][comp] + 8.0 * g.standard_normal((n, d)))
        np.clip(x, 0.0, 255.0, out=x)
        return x.astype(np.uint8)
    raise ValueError(cfg.gen)


def raw_dtype(cfg: Config):
    return np.uint8 if cfg.raw_dtype == "u8" else np.float32


def generate_data(cfg: Config) -> np.ndarray:
    """Database [N x d] (fp32, or uint8 for C5), deterministic in cfg.seed."""
    st = streams(cfg.seed)
    S = _structure(cfg, st)
    nchunks = (cfg.N + CHUNK - 1) // CHUNK
    kids = st["data"].spawn(nchunks)
    out = np.empty((cfg.N, cfg.d), dtype=raw_dtype(cfg))
    for c in range(nchunks):
        lo, hi = c * CHUNK, min(cfg.N, (c + 1) * CHUNK)
        out[lo:hi] = _draw(cfg, S, rng(kids[c]), hi - lo)
    return out


def generate_queries(cfg: Config, nq: int | None = None) -> np.ndarray:
    """Held-out queries [nq x d] fp32 from the same process (uint8-valued for C5)."""
    nq = cfg.nq if nq is None else nq
    st = streams(cfg.seed)
    S = _structure(cfg, st)
    blk = 256   # blocks of 256 queries, each from its own child stream: prefix-stable in nq
    nb = (nq + blk - 1) // blk
    kids = st["queries"].spawn(max(nb, 1))
    q = np.empty((nq, cfg.d), dtype=np.float32)
    for b in range(nb):
        lo, hi = b * blk, min(nq, (b + 1) * blk)
        q[lo:hi] = _draw(cfg, S, rng(kids[b]), blk)[: hi - lo]
    return q
