# C5 (100M x 128 uint8, query-order re-rank): the bench line with the final kernels, then the same
# with Algorithm 4.  Usage (under gpurun): bash tools/c5_ab.sh <tag>
t=${1:-r2c5}
o=gpurun_out
python bench.py --workload C5 --steps 10 --warmup 3 > $o/${t}_bench_c5.json 2> $o/${t}_bench_c5.err
python bench.py --workload C5 --early-rerank --steps 10 --warmup 3 > $o/${t}_bench_c5_alg4.json 2> $o/${t}_bench_c5_alg4.err
tail -c 600 $o/${t}_bench_c5.err
