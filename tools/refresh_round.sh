# Round-end evidence refresh: bench lines for every config, the reference arm,
# launch lists (ncu gpu__time_duration) for c2/c4/c5, one ncu --set full of the
# c4 plane kernel (summarised on the box).  Output: gpurun_out/final_*
set -x
O=gpurun_out
summ() {
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/$1.ncu-rep 25 > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/final_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.txt 2>&1
for c in c2 c1 c3 c4; do
  python bench.py --config $c > $O/final_bench_$c.json 2> $O/final_bench_$c.err
done
python bench.py --config c5 --steps 3 --warmup 3 > $O/final_bench_c5.json 2> $O/final_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/final_bench_ref_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/final_ncu_c2l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_c4_launches.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/final_ncu_c4l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/final_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/final_ncu_c5l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_planes" -s 9 -c 1 -o $O/final_c4_planes python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/final_ncu_c4f.log 2>&1
summ final_c4_planes
du -sh $O
