# Round-end evidence refresh: GPU tests, smoke, bench lines for every config and
# the reference arm (tools/refresh_bench.sh), then timed-region launch lists and
# the c4 plane-kernel ncu capture (tools/launch_lists.sh).  Output: gpurun_out/
set -x
python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1
bash tools/refresh_bench.sh
bash tools/launch_lists.sh
du -sh gpurun_out
