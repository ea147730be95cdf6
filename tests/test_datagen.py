"""Pins of the seeded-input layer: generators, deterministic index build, index file format."""
import os

import numpy as np

import datagen
from datagen import build_index, configs, index_file, synth


def test_generators_deterministic_and_shaped():
    for name in ("C1", "C2", "C3", "C4", "C5"):
        cfg = configs.get(name).replace(N=3000)
        a = synth.generate_data(cfg)
        b = synth.generate_data(cfg)
        assert a.tobytes() == b.tobytes()
        assert a.shape == (3000, cfg.d)
        q = synth.generate_queries(cfg, 300)
        assert np.array_equal(q[:40], synth.generate_queries(cfg, 40))   # prefix-stable
        if name == "C2":
            assert a.min() >= 0 and a.max() <= 255 and np.all(a == np.floor(a))
            assert 10 < a[:, :64].mean() < 40                            # exponential, mean ~20
            assert (a[:, 64:] == 0).mean() > 0.7                          # sparse half
        if name == "C4":
            np.testing.assert_allclose(np.linalg.norm(a, axis=1), 1.0, rtol=1e-5)
        if name == "C5":
            assert a.dtype == np.uint8
        if name == "C3":
            assert 0.3 < a.mean() < 0.7


def test_index_build_partition_and_assignment(c1t):
    cfg, ix, Q, path = c1t
    off = np.asarray(ix["list_offsets"])
    ids = np.asarray(ix["ids"])
    assert off[0] == 0 and off[-1] == cfg.N and np.all(np.diff(off) >= 0)
    assert np.array_equal(np.sort(ids), np.arange(cfg.N))                # a partition
    X = synth.generate_data(cfg)
    raw = np.asarray(ix["raw"])
    assert np.array_equal(raw, X[ids])
    C = np.asarray(ix["centroids"]).astype(np.float64)
    d = ((X[ids].astype(np.float64)[:, None, :] - C[None]) ** 2).sum(2)
    lab = np.repeat(np.arange(cfg.nlist), np.diff(off))
    chosen = d[np.arange(cfg.N), lab]
    assert np.all(chosen <= d.min(1) * (1 + 1e-5) + 1e-6)                # argmin up to near-ties
    for L in range(cfg.nlist):                                            # (list id, point id) order
        seg = ids[off[L]:off[L + 1]]
        assert np.all(np.diff(seg) > 0)


def test_pq_codes_are_nearest_codewords(c1t):
    cfg, ix, Q, _ = c1t
    books = np.asarray(ix["codebooks"]).astype(np.float64)
    codes = np.asarray(ix["codes"])
    raw = np.asarray(ix["raw"]).astype(np.float64)
    ds = cfg.dsub
    for m in range(cfg.M):
        sub = raw[:, m * ds:(m + 1) * ds]
        d = ((sub[:, None, :] - books[m][None]) ** 2).sum(2)
        chosen = d[np.arange(len(sub)), codes[:, m]]
        assert np.all(chosen <= d.min(1) * (1 + 1e-4) + 1e-5)


def test_index_file_roundtrip(tmp_path, c3s):
    cfg, ix, Q, path = c3s
    p = os.path.join(tmp_path, "x.bbcivf")
    index_file.write(p, {k: (np.asarray(v) if hasattr(v, "shape") else v) for k, v in ix.items()})
    ix2 = index_file.read(p, mmap=False)
    for k in ("centroids", "list_offsets", "ids", "P", "wL", "bits", "factors", "raw"):
        assert np.array_equal(np.asarray(ix[k]), ix2[k]), k
    assert ix2["D"] == 960 and ix2["kind"] == "rabitq"


def test_index_cache_key_covers_config():
    a = datagen.index_path(configs.get("C1t"))
    assert a == datagen.index_path(configs.get("C1t").replace(nprobe=7, k=5, budget=9))
    assert a != datagen.index_path(configs.get("C1t").replace(nlist=33))
