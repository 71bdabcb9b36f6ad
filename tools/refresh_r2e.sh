# Round-2 final evidence (fourth session: 2-row groups for the wide plane variants, trimmed resize):
# GPU tests, smoke, bench lines for every config, the reference arm, the 64-frame shard, the c2 / c4
# timed-region launch lists and one ncu --set full of the c2 plane kernel.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/r2f_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/r2f_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2f_smoke.txt 2>&1
for c in c2 c1 c3 c4; do python bench.py --config $c > $O/r2f_bench_$c.json 2> $O/r2f_bench_$c.err; done
python bench.py --config c5 --steps 5 --warmup 3 > $O/r2f_bench_c5.json 2> $O/r2f_bench_c5.err
python bench.py --config c2 --shard-of 8 --no-cpu-baseline > $O/r2f_bench_c2_shard_of_8.json 2> $O/r2f_bench_c2_shard.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/r2f_bench_ref_c2.json 2>&1
for c in c2 c4; do
  ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r2f_${c}_launches.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2f_tl_$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_planes -c 1 -o $O/r2f_planes \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2f_ncu_planes.log 2>&1
python tools/ncu_summary.py $O/r2f_planes.ncu-rep 30 > $O/r2f_planes_summary.txt 2>&1
rm -f $O/r2f_planes.ncu-rep
