# Algorithm 4 (bbc_set_early_rerank) against Algorithm 1 on C2 and C4: parity tests, then the bench
# lines of both.  Usage (under gpurun): bash tools/alg4_ab.sh <tag>
t=${1:-r2i}
o=gpurun_out
python -m pytest tests/test_alg4_gpu.py tests/test_bounds_checks.py -m gpu -q > $o/${t}_alg4.log 2>&1; echo rc=$? >> $o/${t}_alg4.log
for w in C2 C4; do
  python bench.py --workload $w --early-rerank --steps 20 --warmup 5 > $o/${t}_bench_${w,,}_alg4.json 2> $o/${t}_bench_${w,,}_alg4.err
  python bench.py --workload $w --steps 20 --warmup 5 > $o/${t}_bench_${w,,}_alg1.json 2> $o/${t}_bench_${w,,}_alg1.err
done
tail -3 $o/${t}_alg4.log
