set -x
for v in "6 4" "6 3" "4 4" "4 6"; do set -- $v; BBC_LIB_OUT=/tmp/lib_$1_$2.so BBC_NVCC_DEFS="-DBBC_RQ_GPL=$1 -DBBC_RQ_DEPTH=$2" python -c "
import sys; sys.path.insert(0,'.')
from paper_2604_01960_b200 import build; build.build(force=True)"; done
python tools/stage_times.py --workload C4 --nprobe 768 --budget 87500 --steps 3 --tag base_8_2
for v in "6 4" "6 3" "4 4" "4 6"; do set -- $v; BBC_LIB=/tmp/lib_$1_$2.so python tools/stage_times.py --workload C4 --nprobe 768 --budget 87500 --steps 3 --tag v_$1_$2; done
python tools/stage_times.py --workload C4 --nprobe 768 --budget 87500 --steps 3 --tag base_8_2_again
python tools/stage_times.py --workload C2 --nprobe 768 --budget 20000 --steps 5 --tag base_8_2
for v in "6 4" "4 4"; do set -- $v; BBC_LIB=/tmp/lib_$1_$2.so python tools/stage_times.py --workload C2 --nprobe 768 --budget 20000 --steps 5 --tag v_$1_$2; done
