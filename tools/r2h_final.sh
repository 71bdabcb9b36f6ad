# Final tree check: full GPU suite, smoke, default bench line, reference arm, c5 line.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/r2h_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2h_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2h_smoke.txt 2>&1
python bench.py > $O/r2h_bench_default.json 2> $O/r2h_bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/r2h_bench_ref.json 2>&1
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2h_bench_c5.json 2> $O/r2h_bench_c5.err
python bench.py --config c3 --no-cpu-baseline > $O/r2h_bench_c3.json 2> $O/r2h_bench_c3.err
