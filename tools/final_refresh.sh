# Round-end refresh on one B200: GPU tests, smoke, the bench lines, the C4 launch list and an
# ncu --set full capture of the C4 main scan pass.
# Usage (from the repo root, under gpurun): bash tools/final_refresh.sh <tag> [with-c5]
t=${1:-r2f}
o=gpurun_out
python -m pytest tests -m gpu -q --durations=10 > $o/${t}_gputest.log 2>&1; echo rc=$? >> $o/${t}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/${t}_smoke.log 2>&1; echo rc=$? >> $o/${t}_smoke.log
python bench.py --steps 20 --warmup 5 > $o/${t}_bench_c4.json 2> $o/${t}_bench_c4.err
python bench.py --impl reference --steps 3 --warmup 3 > $o/${t}_reference_c4.json 2> $o/${t}_reference_c4.err
for w in C2 C3 C4ip C2q4; do python bench.py --workload $w --steps 20 --warmup 5 > $o/${t}_bench_${w,,}.json 2> $o/${t}_bench_${w,,}.err; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $o/${t}_launches_c4.csv python bench.py --profile-steps --steps 1 --warmup 0 > $o/${t}_ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pq_scan_rq --launch-skip 1 --launch-count 1 \
    -o $o/${t}_scan_c4 python bench.py --profile-steps --steps 1 --warmup 0 > $o/${t}_ncu_scan.log 2>&1
ncu -i $o/${t}_scan_c4.ncu-rep --page raw --csv > $o/${t}_scan_c4_raw.csv 2>/dev/null
rm -f $o/${t}_scan_c4.ncu-rep
if [ -n "$2" ]; then python bench.py --workload C5 --steps 10 --warmup 3 > $o/${t}_bench_c5.json 2> $o/${t}_bench_c5.err; fi
