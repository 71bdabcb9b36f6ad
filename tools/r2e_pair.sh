# 256-bit plane stores by lane pairs (K2_PAIR256): parity under the variant library, then A/B on c3 / c5.
O=gpurun_out
HOGB200_LIB=build/libhog_pair.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_sweep.py tests/test_gpu_slab.py -x -q > $O/r2e_pair_tests.log 2>&1; echo "rc=$?" >> $O/r2e_pair_tests.log
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_pair.so -- c3 c5 > $O/r2e_pair_ab.txt 2>&1
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so@HOGB200_ROWBULK=0 build/libhog_pair.so@HOGB200_ROWBULK=0 -- c2 > $O/r2e_pair_ab_c2.txt 2>&1
