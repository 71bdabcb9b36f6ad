# Integer-tensor-core scores: parity first, then throughput probe, bench lines and a c5 launch list.
O=gpurun_out
./build/probe_imma > $O/r2d_probe_imma.txt 2>&1
python -m pytest tests/test_gpu_scores_i8.py -x -q > $O/r2d_i8_tests.log 2>&1; echo "rc=$?" >> $O/r2d_i8_tests.log
python -m pytest tests -m gpu -x -q > $O/r2d_gpu_tests2.log 2>&1; echo "tests rc=$?" >> $O/r2d_gpu_tests2.log
for c in c4 c1; do python bench.py --config $c --no-cpu-baseline > $O/r2d_bench_$c.json 2> $O/r2d_bench_$c.err; done
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2d_bench_c5_i8.json 2> $O/r2d_bench_c5_i8.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r2d_c5_launches_i8.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2d_tl_c5_i8.log 2>&1
