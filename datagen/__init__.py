"""Seeded-input layer shared by the oracle, the tests and bench.py.

Holds the workload configs, the seeded synthetic generators, the deterministic index builder and
the index-file format.  It contains none of the BBC query-path arithmetic (probe, LUT, estimate,
buckets, threshold, compaction, re-rank, select): that lives twice, independently, in `oracle/`
(CPU reference) and in `paper_2604_01960_b200/csrc/` (CUDA).
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

from . import build_index, configs, index_file, synth  # noqa: F401
from .configs import Config, get  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))


def _source_hash() -> str:
    h = hashlib.sha1()
    for fn in ("configs.py", "synth.py", "build_index.py", "index_file.py"):
        with open(os.path.join(_HERE, fn), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:12]


def cache_dir() -> str:
    d = os.environ.get("BBC_CACHE", "/tmp/bbc_cache")
    os.makedirs(d, exist_ok=True)
    return d


_BUILD_FIELDS = ("gen", "N", "d", "raw_dtype", "kind", "nlist", "M", "seed", "kmeans_iters",
                 "kmeans_train_per_list", "pq_train", "pq_iters", "metric", "pq_bits")


def index_path(cfg: Config) -> str:
    """Cache path keyed by the build-relevant fields of cfg and this package's sources."""
    desc = repr(tuple(getattr(cfg, f) for f in _BUILD_FIELDS))
    key = hashlib.sha1(desc.encode() + _source_hash().encode()).hexdigest()[:12]
    return os.path.join(cache_dir(), f"{cfg.name}_{key}.bbcivf")


def _drop_stale(path: str, cfg: Config) -> None:
    """Delete cached index files of the same workload built from other sources or settings (a
    full-size index is up to 17 GB; a long-lived cache directory would otherwise fill the disk)."""
    d, base = os.path.split(path)
    prefix = f"{cfg.name}_"
    try:
        for fn in os.listdir(d):
            if fn.startswith(prefix) and fn.endswith(".bbcivf") and fn != base:
                full = os.path.join(d, fn)
                if os.path.getsize(full) > (256 << 20):      # only the big full-size files
                    os.remove(full)
    except OSError:
        pass


def ensure_index(cfg: Config, verbose: bool = False) -> str:
    """Path of cfg's serialized index, building it (deterministically from the seed) if absent.

    The cache key covers the config and this package's sources, so a stale file is never reused.
    """
    path = index_path(cfg)
    if not os.path.exists(path):
        _drop_stale(path, cfg)
        t0 = time.time()
        idx = build_index.build(cfg, verbose=verbose)
        index_file.write(path, idx)
        if verbose:
            print(f"[datagen] built {cfg.name} index in {time.time() - t0:.1f}s -> {path}", file=sys.stderr)
    return path
