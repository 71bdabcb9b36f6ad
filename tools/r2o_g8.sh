# 2-row groups for the 8-columns-per-lane plane variants: full GPU suite, then c4 / c2 / c1 bench lines.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/r2o_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2o_gpu_tests.log
for c in c4 c2 c1; do python bench.py --config $c --no-cpu-baseline > $O/r2o_bench_$c.json 2> $O/r2o_bench_$c.err; done
