# re-rank tuning for <= 512-byte rows: CTAs per SM (BBC_RR_MINB512) and rows in flight per lane
# group (BBC_RR_STEPS512); default 4 x 1
for v in "5 1" "6 1" "4 2"; do set -- $v; BBC_LIB_OUT=/tmp/lib_rr_$1_$2.so BBC_NVCC_DEFS="-DBBC_RR_MINB512=$1 -DBBC_RR_STEPS512=$2" python -c "
import sys; sys.path.insert(0,'.')
from paper_2604_01960_b200 import build; build.build(force=True)"; done
for w in "C4 768 85000 3" "C2 768 20000 5"; do set -- $w
  python tools/stage_times.py --workload $1 --nprobe $2 --budget $3 --steps $4 --tag rr_4_1
  for v in "5 1" "6 1" "4 2"; do set -- $w; a=$1; b=$2; c=$3; d=$4; set -- $v; BBC_LIB=/tmp/lib_rr_$1_$2.so python tools/stage_times.py --workload $a --nprobe $b --budget $c --steps $d --tag rr_$1_$2; done
done
