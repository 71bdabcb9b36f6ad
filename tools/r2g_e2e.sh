# New e2e chunking default (a quarter of the step's frames per chunk): bench lines, multirank gather test.
O=gpurun_out
python -m pytest tests/test_gpu_multirank.py -x -q > $O/r2g_multirank.log 2>&1; echo "rc=$?" >> $O/r2g_multirank.log
for rep in 1 2 3; do python bench.py --config c2 > $O/r2g_bench_c2_$rep.json 2> $O/r2g_bench_c2_$rep.err; done
python bench.py --config c2 --e2e-chunk 64 --e2e-slots 8 --no-cpu-baseline > $O/r2g_bench_c2_64x8.json 2> $O/r2g_bench_c2_64x8.err
for c in c1 c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/r2g_bench_$c.json 2> $O/r2g_bench_$c.err; done
python bench.py --config c2 --shard-of 8 --no-cpu-baseline > $O/r2g_shard8.json 2> $O/r2g_shard8.err
