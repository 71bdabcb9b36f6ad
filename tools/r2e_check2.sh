# Random sweep + full GPU suite + c5/c3 bench with 2-row groups and the trimmed resize.
O=gpurun_out
python -m pytest tests/test_gpu_random_sweep.py -q > $O/r2e_sweep.log 2>&1; echo "rc=$?" >> $O/r2e_sweep.log
python -m pytest tests -m gpu -q -x > $O/r2e_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2e_gpu_tests.log
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2e_bench_c5b.json 2> $O/r2e_bench_c5b.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r2e_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2e_tl_c5.log 2>&1
