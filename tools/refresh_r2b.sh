# Round-2 (second session) evidence: GPU tests, smoke, bench lines for every
# config, the reference arm, the 64-frame shard, and the c2 timed-region launch list.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/r2b_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2b_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2b_smoke.txt 2>&1
for c in c2 c1 c3 c4; do python bench.py --config $c > $O/r2b_bench_$c.json 2> $O/r2b_bench_$c.err; done
python bench.py --config c5 --steps 3 --warmup 3 > $O/r2b_bench_c5.json 2> $O/r2b_bench_c5.err
python bench.py --config c2 --shard-of 8 --no-cpu-baseline > $O/r2b_bench_c2_shard_of_8.json 2> $O/r2b_bench_c2_shard.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/r2b_bench_ref_c2.json 2>&1
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r2b_c2_launches.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2b_tl_c2.log 2>&1
