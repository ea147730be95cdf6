"""Per-kernel registers / spills from `nvcc -Xptxas -v` output of the library build."""
import re
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2604_01960_b200 import build as B  # noqa: E402

nccl = B._nccl_dir()
cmd = [B.NVCC, *B.FLAGS, "-I", B.os.path.join(B.ROOT, "include"), "-I", B.os.path.join(nccl, "include"),
       *B.SOURCES, "-o", "/tmp/ptxas_probe.so", "-lcudart", "-L", B.os.path.join(nccl, "lib"), "-l:libnccl.so.2"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        if pat in cur:
            print(f"{int(m2.group(1)):4d} regs spill {spill[0]:4d}/{spill[1]:4d}  {cur[:150]}")
        cur = None
