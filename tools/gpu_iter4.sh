set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/gpu_tests4.log 2>&1
for c in c2 c4 c3; do python bench.py --config $c --no-cpu-baseline > $O/t4_$c.json 2> $O/t4_$c.err; done
python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > $O/t4_c5.json 2> $O/t4_c5.err
