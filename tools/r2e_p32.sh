# Row-bulk plane kernel with full 32-bit register state (K2_RB_P32): parity, then A/B against the packed form.
O=gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_kats.py tests/test_gpu_slab.py tests/test_gpu_resize.py -x -q > $O/r2e_p32_tests.log 2>&1; echo "rc=$?" >> $O/r2e_p32_tests.log
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_p32off.so -- c2 c2:--shard-of=8 c1 > $O/r2e_p32_ab.txt 2>&1
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r2e_bench_c5.json 2> $O/r2e_bench_c5.err
