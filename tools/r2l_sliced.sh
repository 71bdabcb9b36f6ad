# Bit-sliced column counts in the gather binning kernel (K1_SLICED): parity, then A/B on c3 / c5.
O=gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_slab.py tests/test_gpu_pyramid.py tests/test_gpu_c5_full.py tests/test_gpu_octant.py -x -q > $O/r2l_tests.log 2>&1; echo "rc=$?" >> $O/r2l_tests.log
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_unsliced.so -- c3 c5 > $O/r2l_ab.txt 2>&1
