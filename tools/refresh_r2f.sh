# Final evidence after the carry-scan fold: bench lines, launch lists, c2 plane-kernel ncu.
O=gpurun_out
for c in c1 c3 c4; do python bench.py --config $c > $O/r2s_bench_$c.json 2> $O/r2s_bench_$c.err; done
python bench.py --config c5 --steps 5 --warmup 3 > $O/r2s_bench_c5.json 2> $O/r2s_bench_c5.err
python bench.py --config c2 --shard-of 8 --no-cpu-baseline > $O/r2s_bench_c2_shard_of_8.json 2> $O/r2s_shard.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/r2s_bench_ref_c2.json 2>&1
for c in c2 c4; do
  ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/r2s_${c}_launches.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2s_tl_$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_planes -c 1 -o $O/r2s_planes \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/r2s_ncu_planes.log 2>&1
python tools/ncu_summary.py $O/r2s_planes.ncu-rep 30 > $O/r2s_planes_summary.txt 2>&1
rm -f $O/r2s_planes.ncu-rep
