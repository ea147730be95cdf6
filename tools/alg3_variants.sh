# Algorithm 3 kernel (k_alg3) variants on C3 at eps0 1.3: rows per warp in flight (BBC_A3_NR) x
# vectors per lane per round (BBC_A3_V) x CTAs per SM (BBC_A3_MINB); default 2 x 2 x 2 (first sweep: profiles/r02_alg3_variants_c3.log)
V="${A3V:-1_8_2 2_4_2 2_2_2 4_2_2 1_4_2 2_4_1 4_4_1}"
# build (here, cross-compiling) with "build", run (on the GPU box) with "run"
mkdir -p build_variants
[ "$1" = build ] && for v in $V; do IFS=_ read nr vv mb <<< "$v"; BBC_LIB_OUT=build_variants/lib_a3_$v.so BBC_NVCC_DEFS="-DBBC_A3_NR=$nr -DBBC_A3_V=$vv -DBBC_A3_MINB=$mb" python -c "
import sys; sys.path.insert(0,'.')
from paper_2604_01960_b200 import build; build.build(force=True)" || exit 1; done
[ "$1" = run ] && for v in $V; do BBC_LIB=build_variants/lib_a3_$v.so python tools/stage_times.py --workload C3 --nprobe 2048 --budget 20000 --steps 3 --bound-rerank 1.3 --gathers query --tag a3_$v; done
