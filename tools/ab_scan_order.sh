# usage: bash ab.sh tag
t=$1
W=${2:-C4}; NP=${3:-768}; BU=${4:-85000}
for o in probe sweep probe sweep; do python tools/stage_times.py --workload $W --nprobe $NP --budget $BU --ws-gb 96 --order $o --tag $o --steps 5; done > gpurun_out/${t}_stages.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_pq_scan_rq --launch-count 2 --csv --log-file gpurun_out/${t}_ncu_sweep.csv python tools/stage_times.py --workload $W --nprobe $NP --budget $BU --ws-gb 96 --order sweep --steps 1 > /dev/null 2>&1
python - <<PY
import csv, json
for l in open("gpurun_out/${t}_stages.jsonl"):
    try:
        d = json.loads(l); print(d["tag"], round(d["ms_per_step"],2), "sample", d["sample"], "scan", d["scan"])
    except Exception: print(l.strip()[:200])
rows=[r for r in csv.reader(open("gpurun_out/${t}_ncu_sweep.csv")) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d["Kernel Name"][:26], d["Metric Name"], d["Metric Value"])
PY
