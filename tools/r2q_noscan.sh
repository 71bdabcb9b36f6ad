# Carry scan folded into the plane kernel for few-band shapes (HOGB200_NOSCAN_PCT): parity, then A/B.
O=gpurun_out
python -m pytest tests -m gpu -q -x > $O/r2q_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2q_gpu_tests.log
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so paper_1703_06256_b200/libhogb200.so@HOGB200_NOSCAN_PCT=0 paper_1703_06256_b200/libhogb200.so@HOGB200_NOSCAN_PCT=30 -- c1 c4 c3 > $O/r2q_ab2.txt 2>&1
python bench.py --config c2 > $O/r2q_bench_c2.json 2> $O/r2q_bench_c2.err
