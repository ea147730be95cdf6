# ncu of Algorithm 4's kernels on C4 (one micro-batch step): launch list with DRAM bytes, then a
# --set full capture of k_early_rows.  Usage (under gpurun): bash tools/alg4_ncu.sh <tag>
t=${1:-r2n}
o=gpurun_out
python bench.py --early-rerank --profile-steps --steps 1 --warmup 0 > $o/${t}_alg4_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $o/${t}_launches_c4_alg4.csv python bench.py --early-rerank --profile-steps --steps 1 --warmup 0 > $o/${t}_ncu_alg4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_early_rows --launch-skip 1 --launch-count 1 \
    -o $o/${t}_early_c4 python bench.py --early-rerank --profile-steps --steps 1 --warmup 0 > $o/${t}_ncu_early.log 2>&1
ncu -i $o/${t}_early_c4.ncu-rep --page raw --csv > $o/${t}_early_c4_raw.csv 2>/dev/null
rm -f $o/${t}_early_c4.ncu-rep
