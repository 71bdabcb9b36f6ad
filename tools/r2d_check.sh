# Round-2 re-entry check: GPU tests, smoke, c2 bench, and a c5 timed-region launch list.
O=gpurun_out
python -m pytest tests -m gpu -q -x > $O/r2d_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2d_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2d_smoke.txt 2>&1
python bench.py --config c2 > $O/r2d_bench_c2.json 2> $O/r2d_bench_c2.err
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2d_bench_c5.json 2> $O/r2d_bench_c5.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r2d_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2d_tl_c5.log 2>&1
