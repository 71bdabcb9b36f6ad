# resize parity + c5 plane-kernel source-level profile + c5 bench with the row-shared resize
O=gpurun_out
python -m pytest tests/test_gpu_resize.py tests/test_gpu_parity.py -k "resize or pyramid" -x -q > $O/r2d_resize_tests.log 2>&1; echo "rc=$?" >> $O/r2d_resize_tests.log
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2d_bench_c5_rz.json 2> $O/r2d_bench_c5_rz.err
HOGB200_RESIZE_ROWS=0 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/r2d_bench_c5_rz0.json 2> $O/r2d_bench_c5_rz0.err
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r2d_c5_launches_rz.csv python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2d_tl_c5_rz.log 2>&1
bash tools/c5_planes_profile.sh
