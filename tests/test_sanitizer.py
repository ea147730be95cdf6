"""compute-sanitizer over one small search per index kind: memcheck (out-of-bounds
and misaligned accesses), racecheck (shared-memory hazards) and synccheck (barrier misuse) on
the PQ path (replicated-LUT scan, compaction, re-rank, select; C1t) and the RaBitQ tensor-core
path (TMA, mbarriers, tcgen05/TMEM GEMM; C3s).  Each run is a subprocess under the tool with
--error-exitcode, so any reported hazard fails the test."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("name,nprobe,budget,nq", [("C1t", 6, 600, 4), ("C3s", 12, 1500, 4)])
def test_compute_sanitizer(tool, name, nprobe, budget, nq, load):
    load(name)                                            # index file built outside the tool
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "one_search.py"), "--workload", name,
           "--nprobe", str(nprobe), "--budget", str(budget), "--reps", "1", "--nq", str(nq)]
    if tool == "memcheck":
        cmd[3:3] = ["--leak-check", "no"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr or "RACECHECK SUMMARY: 0 hazards" in r.stdout + r.stderr, tail
