# CTAs per SM of the <= 512-byte-row re-rank kernels (BBC_RR_MINB512): 4 (default) vs 5, 6
for m in 5 6; do BBC_LIB_OUT=/tmp/lib_rr$m.so BBC_NVCC_DEFS="-DBBC_RR_MINB512=$m" python -c "
import sys; sys.path.insert(0,'.')
from paper_2604_01960_b200 import build; build.build(force=True)"; done
python tools/stage_times.py --workload C4 --nprobe 768 --budget 87500 --steps 3 --tag rr4
for m in 5 6; do BBC_LIB=/tmp/lib_rr$m.so python tools/stage_times.py --workload C4 --nprobe 768 --budget 87500 --steps 3 --tag rr$m; done
python tools/stage_times.py --workload C2 --nprobe 768 --budget 20000 --steps 5 --tag rr4
for m in 5 6; do BBC_LIB=/tmp/lib_rr$m.so python tools/stage_times.py --workload C2 --nprobe 768 --budget 20000 --steps 5 --tag rr$m; done
