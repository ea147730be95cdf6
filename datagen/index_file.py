"""Serialized IVF index file ("BBCIVF01") -- the contract between index build and both query paths.

Layout (little-endian; DESIGN.md section 4 is the normative copy, `include/bbc.h` repeats it):

  bytes [0, 8)      magic  b"BBCIVF01"
  bytes [8, 256)    31 x int64 header fields:
                      0 version(=1)  1 kind(1=PQ, 2=RaBitQ)  2 raw_dtype(0=f32, 1=u8)
                      3 N  4 d  5 nlist  6 M  7 nbits  8 D  9 seed  10 n_sections(=10)
                      11 metric (0 = squared L2, 1 = inner product; keys are -<q, x>)
  bytes [256, 416)  section table: 10 x (int64 offset, int64 nbytes); offset 0 = absent
  sections, each 256-byte aligned, in this order:
      0 centroids    f32 [nlist x d]
      1 list_offsets i64 [nlist + 1]          (list L = rows [off[L], off[L+1]) of the list-ordered arrays)
      2 ids          i64 [N]                  (original id of each list-ordered row)
      3 codebooks    f32 [M x 2^nbits x d/M]  (PQ only; nbits 8 or 4)
      4 codes        u8  [N x M]              (PQ only, list order; one code per byte)
      5 P            f32 [D x D]              (RaBitQ only; y = P^T o)
      6 wL           f32 [nlist x D]          (RaBitQ only; w_L = P^T c_L, c_L zero-padded to D)
      7 bits         u8  [N x D/8]            (RaBitQ only; bit i of row in byte i/8, LSB first)
      8 factors      f32 [N x 2]              (RaBitQ only; (r_o, g_o))
      9 raw          f32|u8 [N x d]           (list order)

Seeded-input layer: read/write only, no query arithmetic.
"""
from __future__ import annotations

import os

import numpy as np

MAGIC = b"BBCIVF01"
VERSION = 1
SECTIONS = ("centroids", "list_offsets", "ids", "codebooks", "codes", "P", "wL", "bits",
            "factors", "raw")
KIND = {"pq": 1, "rabitq": 2}
RAW = {"f32": 0, "u8": 1}
METRIC = {"l2": 0, "ip": 1}


def _align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


def write(path: str, idx: dict) -> None:
    kind = KIND[idx["kind"]]
    hdr = np.zeros(31, dtype=np.int64)
    hdr[0] = VERSION
    hdr[1] = kind
    hdr[2] = RAW[idx["raw_dtype"]]
    hdr[3] = idx["N"]
    hdr[4] = idx["d"]
    hdr[5] = idx["nlist"]
    hdr[6] = idx.get("M", 0)
    hdr[7] = idx.get("nbits", 8)
    hdr[8] = idx.get("D", 0)
    hdr[9] = idx.get("seed", 0)
    hdr[10] = len(SECTIONS)
    hdr[11] = METRIC[idx.get("metric", "l2")]
    want = {
        "centroids": np.float32, "list_offsets": np.int64, "ids": np.int64,
        "codebooks": np.float32, "codes": np.uint8, "P": np.float32, "wL": np.float32,
        "bits": np.uint8, "factors": np.float32,
        "raw": np.uint8 if idx["raw_dtype"] == "u8" else np.float32,
    }
    table = np.zeros((len(SECTIONS), 2), dtype=np.int64)
    pos = 512
    arrays = []
    for i, name in enumerate(SECTIONS):
        a = idx.get(name)
        if a is None:
            continue
        a = np.ascontiguousarray(a, dtype=want[name])
        pos = _align(pos)
        table[i] = (pos, a.nbytes)
        arrays.append((pos, a))
        pos += a.nbytes
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(MAGIC)
        f.write(hdr.tobytes())
        f.write(table.tobytes())
        for off, a in arrays:
            f.seek(off)
            f.write(memoryview(a.reshape(-1).view(np.uint8)))
        f.truncate(pos)
    os.replace(tmp, path)


def read(path: str, mmap: bool = True) -> dict:
    with open(path, "rb") as f:
        head = f.read(512)
    if head[:8] != MAGIC:
        raise ValueError(f"{path}: bad magic")
    hdr = np.frombuffer(head[8:256], dtype=np.int64)
    table = np.frombuffer(head[256:256 + 16 * len(SECTIONS)], dtype=np.int64).reshape(-1, 2)
    if hdr[0] != VERSION:
        raise ValueError(f"{path}: version {hdr[0]}")
    kind = {v: k for k, v in KIND.items()}[int(hdr[1])]
    raw_dtype = {v: k for k, v in RAW.items()}[int(hdr[2])]
    N, d, nlist, M, nbits, D, seed = (int(x) for x in hdr[3:10])
    shapes = {
        "centroids": ((nlist, d), np.float32), "list_offsets": ((nlist + 1,), np.int64),
        "ids": ((N,), np.int64), "codebooks": ((M, 1 << nbits if kind == "pq" else 256, d // M if M else 0), np.float32),
        "codes": ((N, M), np.uint8), "P": ((D, D), np.float32), "wL": ((nlist, D), np.float32),
        "bits": ((N, D // 8), np.uint8), "factors": ((N, 2), np.float32),
        "raw": ((N, d), np.uint8 if raw_dtype == "u8" else np.float32),
    }
    metric = {v: k for k, v in METRIC.items()}[int(hdr[11])]
    out = dict(kind=kind, raw_dtype=raw_dtype, N=N, d=d, nlist=nlist, M=M, nbits=nbits, D=D,
               seed=seed, metric=metric)
    for i, name in enumerate(SECTIONS):
        off, nb = (int(x) for x in table[i])
        if off == 0:
            continue
        shape, dt = shapes[name]
        if nb != int(np.prod(shape)) * np.dtype(dt).itemsize:
            raise ValueError(f"{path}: section {name} has {nb} bytes, expected shape {shape}")
        if mmap:
            out[name] = np.memmap(path, dtype=dt, mode="r", offset=off, shape=shape)
        else:
            with open(path, "rb") as f:
                f.seek(off)
                out[name] = np.fromfile(f, dtype=dt, count=int(np.prod(shape))).reshape(shape)
    return out
