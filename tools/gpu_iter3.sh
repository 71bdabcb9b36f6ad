set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/gpu_tests3.log 2>&1
for ch in 1 2 4; do
  HOGB200_CHUNKS=$ch python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/ch_c4_$ch.json 2>&1
  HOGB200_CHUNKS=$ch python bench.py --config c3 --no-cpu-baseline --no-e2e > $O/ch_c3_$ch.json 2>&1
done
HOGB200_CHUNKS=2 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/ch_c2_2.json 2>&1
