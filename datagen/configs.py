"""Workload configurations C1..C5 (BASELINE.json `configs[0..4]`) and scaled test variants.

This module is part of the seeded-input layer (`datagen/`): it holds shapes, seeds and
search parameters only -- none of the method's arithmetic.  Both the oracle (`oracle/`)
and the CUDA path (`paper_2604_01960_b200/`) consume what `datagen` produces.

Sources
  * BASELINE.json configs[0..4]  -> C1..C5 (N, d, storage, quantizer, nlist, nq, k, nprobe,
    budget multiplier).
  * SURVEY.md section 8(d) "Synthetic inputs" -> generator recipes (see `synth.py`).
  * Seeds: base 260401960 + config index (1..5), SURVEY.md 8(d).
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

SEED_BASE = 260401960


@dataclass(frozen=True)
class Config:
    name: str            # "C1" ... "C5" or a scaled variant such as "C2s"
    gen: str             # generator id: "C1".."C5" (the recipe in synth.py)
    N: int               # database size
    d: int               # dimensionality
    raw_dtype: str       # "f32" or "u8" (storage of raw vectors)
    kind: str            # "pq" or "rabitq"
    nlist: int           # IVF lists
    M: int               # PQ sub-quantizers (0 for RaBitQ)
    nq: int              # queries per batch
    k: int               # top-k
    nprobe: int          # lists probed per query
    budget: int          # candidate budget (n_cand in the paper)
    seed: int            # base seed of the generator
    # index-build knobs (deterministic; the serialized file is the contract)
    kmeans_iters: int = 10
    kmeans_train_per_list: int = 64
    pq_train: int = 65536
    pq_iters: int = 12
    metric: str = "l2"   # "l2" (squared L2) or "ip" (inner product, keys -<q,x>)
    pq_bits: int = 8     # bits per PQ sub-quantizer code: 8 (256 centroids) or 4 (16)
    extra: dict = field(default_factory=dict, compare=False, hash=False)

    @property
    def dsub(self) -> int:
        return self.d // self.M if self.M else 0

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs, verbatim shapes.
C1 = Config("C1", "C1", 100_000, 128, "f32", "pq", 256, 16, 100, 5_000, 32, 10_000, SEED_BASE + 1,
            kmeans_iters=20)
C2 = Config("C2", "C2", 1_000_000, 128, "f32", "pq", 4_096, 32, 1_000, 10_000, 128, 20_000,
            SEED_BASE + 2)
C3 = Config("C3", "C3", 1_000_000, 960, "f32", "rabitq", 4_096, 0, 1_000, 5_000, 256, 15_000,
            SEED_BASE + 3)
C4 = Config("C4", "C4", 10_000_000, 96, "f32", "pq", 16_384, 48, 10_000, 50_000, 512, 75_000,
            SEED_BASE + 4)
C5 = Config("C5", "C5", 100_000_000, 128, "u8", "pq", 65_536, 32, 10_000, 20_000, 1_024, 40_000,
            SEED_BASE + 5)

FULL = {c.name: c for c in (C1, C2, C3, C4, C5)}

# Scaled variants used by the parity tests: same generators and structure, sizes the CPU oracle
# finishes in seconds while still spanning many tiles and ragged list tails.
SMALL = {
    "C1t": C1.replace(name="C1t", N=6_000, nlist=32, nq=12, k=300, nprobe=6, budget=600),
    "C1s": C1.replace(name="C1s", nq=24),
    "C2s": C2.replace(name="C2s", N=120_000, nlist=512, nq=24, k=1_500, nprobe=24, budget=3_000,
                      kmeans_iters=8),
    "C3s": C3.replace(name="C3s", N=40_000, nlist=128, nq=12, k=500, nprobe=12, budget=1_500,
                      kmeans_iters=8),
    "C4s": C4.replace(name="C4s", N=200_000, nlist=512, nq=24, k=2_000, nprobe=32, budget=3_000,
                      kmeans_iters=6),
    "C5s": C5.replace(name="C5s", N=200_000, nlist=512, nq=24, k=1_500, nprobe=32, budget=3_000,
                      kmeans_iters=6),
    # RaBitQ at the dimension limits of the tensor-core path: D = 1024 (two B stages, all 512 TMEM
    # columns in use) and D = 64 (one K block, two MMAs per tile)
    "C3d1024s": C3.replace(name="C3d1024s", d=1024, N=20_000, nlist=64, nq=8, k=300, nprobe=10,
                           budget=900, kmeans_iters=6),
    "C3d64s": C3.replace(name="C3d64s", d=64, N=30_000, nlist=96, nq=8, k=300, nprobe=12,
                         budget=900, kmeans_iters=6),
    # d = 200: D = 256 with 56 zero-padded dimensions, d not a multiple of the rotation's 16-row
    # P blocks, 11 queries (the rotation's last CTA holds 3 of its 8)
    "C3d200s": C3.replace(name="C3d200s", d=200, N=20_000, nlist=64, nq=11, k=300, nprobe=10,
                          budget=900, kmeans_iters=6),
    # RaBitQ tensor-core GEMM beyond one query tile per list: every query probes (nearly) every
    # list, so each list's Push pass runs >= 5 query tiles of kRbN = 96 pairs (both TMEM
    # accumulators, the B-stage ring and the 4-deep records ring wrap; the producer loop runs),
    # the sample pass >= 2.  D = 128 keeps the oracle fast; C3mt960 repeats it at C3's D = 960
    # (8 K blocks per B stage).
    "C3mt": C3.replace(name="C3mt", d=128, N=24_000, nlist=16, nq=540, k=300, nprobe=15,
                       budget=900, kmeans_iters=6),
    "C3mt960": C3.replace(name="C3mt960", N=8_000, nlist=8, nq=500, k=200, nprobe=8, budget=600,
                          kmeans_iters=6),
    # the scan's other sub-quantizer counts: M = 64 (dsub 2) and M = 24 (dsub 4), M = 8 (dsub 12)
    "C2m64s": C2.replace(name="C2m64s", M=64, N=60_000, nlist=256, nq=12, k=800, nprobe=16, budget=1_600,
                         kmeans_iters=6),
    "C4m24s": C4.replace(name="C4m24s", M=24, N=60_000, nlist=256, nq=12, k=800, nprobe=16, budget=1_600,
                         kmeans_iters=6),
    "C4m8s": C4.replace(name="C4m8s", M=8, N=60_000, nlist=256, nq=12, k=800, nprobe=16, budget=1_600,
                        kmeans_iters=6),
    # fine lists (~20 objects): a compaction chunk of 8,192 objects spans > 256 lists, the
    # global-search path of k_emit; probe sets of 600 lists
    "C2f": C2.replace(name="C2f", N=40_000, nlist=2_048, nq=8, k=500, nprobe=600, budget=1_000,
                      kmeans_iters=4),
    # Algorithm 3 (f1) on RaBitQ indexes of integer-valued data (C2's generator as fp32, C5's as
    # uint8): exact d^2 are integers < 2^24, identical in fp32 and fp64, so the exact distances'
    # bucket ids that steer Algorithm 3's loop agree on both sides and its re-ranked set is compared
    # exactly.  40 queries over 12 of 64 lists: tensor-core query tiles per list > 1.
    "C3a3": C3.replace(name="C3a3", gen="C2", d=128, N=30_000, nlist=64, nq=40, k=300, nprobe=12,
                       budget=900, kmeans_iters=6),
    "C3a3u8": C3.replace(name="C3a3u8", gen="C5", raw_dtype="u8", d=128, N=30_000, nlist=64, nq=16,
                         k=300, nprobe=12, budget=900, kmeans_iters=6),
    # D = 512 uint8 rows (the u8 limit; 8 K blocks of the RaBitQ GEMM): exact d^2 of the
    # candidates stay integers < 2^24
    "C3a3u8d512": C3.replace(name="C3a3u8d512", gen="C5", raw_dtype="u8", d=512, N=20_000, nlist=48,
                             nq=12, k=200, nprobe=10, budget=600, kmeans_iters=6),
}

# Inner-product / cosine variants ("our result buffer
# applies to ... cosine similarity and inner product"): the C4 generator's vectors are unit norm,
# so inner product = cosine similarity.  The IVF lists are the same L2 k-means lists.
IP = {
    "C4ip": C4.replace(name="C4ip", metric="ip"),
    "C4ip_s": SMALL["C4s"].replace(name="C4ip_s", metric="ip"),
}

# 4-bit PQ, the paper's PQ setting ("M = d/4 ... 4 bits per
# sub-vector, B = d"): C2's data with M = 32 sub-quantizers of 16 centroids (dsub 4), estimated
# with the FastScan-style 8-bit quantised lookup table (reading R20).
PQ4 = {
    "C2q4": C2.replace(name="C2q4", pq_bits=4),
    "C2q4s": SMALL["C2s"].replace(name="C2q4s", pq_bits=4),
}

ALL = {**FULL, **SMALL, **IP, **PQ4}


def get(name: str) -> Config:
    return ALL[name]
