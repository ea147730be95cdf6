"""The bounds-checked build (BBC_CHECKS=1: device-side checks on the indices the PQ scan, its
sweep-order kernels, the compaction, the selections and Algorithm 3's kernel compute; a violation traps) runs the
search paths without a trap and returns the default build's results bit for bit.

compute-sanitizer is closed on the GPU pool, so this stands in for memcheck on those kernels.
Each library runs in its own process (the binding loads one library per process, chosen by
BBC_LIB)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (config, k, nprobe, budget, scan order): probe and sweep order (with the sample pass filled
# up), a main pass with no lists (nprobe 1), tau = infinity, every list probed, the list-sharded
# group search
CASES = [("C1t", None, None, None, "probe"), ("C1t", None, None, None, "sweep"),
         ("C1t", 5000, 1, 5000, "sweep"), ("C1t", 300, 32, 600, "sweep"),
         ("C2s", None, None, None, "sweep"), ("C4s", None, None, None, "sweep"),
         ("C4s", None, None, None, "probe"), ("C5s", None, None, None, "sweep"),
         ("C4ip_s", None, None, None, "sweep"), ("C2s", None, None, None, "group-sweep"),
         ("C3a3", None, None, None, "alg3"), ("C3a3u8", None, None, None, "alg3"),
         ("C3a3", None, 3, 10 ** 6, "alg3"),    # Algorithm 3 (f1): finite tau, uint8 rows, no sample
         ("C2s", None, 12, 18_000, "alg4"), ("C5s", None, 12, 30_000, "alg4"),   # Algorithm 4 (f2): many
         ("C4ip_s", None, None, None, "alg4")]                                   # early objects; uint8; IP

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import datagen
from datagen import configs, synth
from paper_2604_01960_b200 import Index
from paper_2604_01960_b200.bbc import search_group
out = {}
for i, (name, k, nprobe, budget, order) in enumerate(json.loads(sys.argv[2])):
    cfg = configs.get(name)
    path = datagen.ensure_index(cfg)
    k, nprobe, budget = k or cfg.k, nprobe or cfg.nprobe, budget or cfg.budget
    q = torch.from_numpy(synth.generate_queries(cfg)).cuda()
    if order == "group-sweep":
        shards = [Index(path, rank=r, world=2) for r in range(2)]
        for s in shards:
            s.set_scan_order(s.ORDER_SWEEP)
        ids, d2 = search_group(shards, q, k, nprobe, budget)
    elif order == "alg3":
        g = Index(path)
        g.set_bound_rerank(True, 1.2)
        ids, d2 = g.search(q, k, nprobe, budget)
        o = torch.argsort(ids, dim=1)                 # candidate order unspecified: sort by id
        ids, d2 = ids.gather(1, o), d2.gather(1, o)
    elif order == "alg4":
        g = Index(path)
        g.set_early_rerank(True)
        ids, d2 = g.search(q, k, nprobe, budget)
    else:
        g = Index(path)
        g.set_scan_order(g.ORDER_SWEEP if order == "sweep" else g.ORDER_PROBE)
        ids, d2 = g.search(q, k, nprobe, budget)
    torch.cuda.synchronize()
    out[f"ids{i}"] = ids.cpu().numpy()
    out[f"d2{i}"] = d2.cpu().numpy()
np.savez(sys.argv[3], **out)
from paper_2604_01960_b200 import bbc
print("ok", bbc.lib()._name)
"""


def _run(lib, dst):
    env = dict(os.environ)
    if lib:
        env["BBC_LIB"] = lib
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, json.dumps(CASES), dst], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    if lib:                                           # the checked library is the one that ran
        assert r.stdout.strip().split()[-1] == lib, r.stdout[-500:]


def test_bounds_checked_build_matches_default(tmp_path):
    lib = str(tmp_path / "libbbc_checks.so")
    env = dict(os.environ, BBC_LIB_OUT=lib, BBC_NVCC_DEFS="-DBBC_CHECKS=1")
    r = subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, sys.argv[1]); "
                        "from paper_2604_01960_b200 import build; build.build(force=True)", ROOT],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    _run(lib, str(tmp_path / "checked.npz"))
    _run(None, str(tmp_path / "default.npz"))
    a, b = np.load(tmp_path / "checked.npz"), np.load(tmp_path / "default.npz")
    for key in a.files:
        assert np.array_equal(a[key], b[key]), key
