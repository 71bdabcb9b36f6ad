set -x
O=gpurun_out
summ() {
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/$1.ncu-rep 25 > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
python bench.py --config c4 --no-cpu-baseline > $O/it2_c4.json 2> $O/it2_c4.err
python bench.py --config c1 --no-cpu-baseline > $O/it2_c1.json 2> $O/it2_c1.err
python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > $O/it2_c5.json 2> $O/it2_c5.err
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows" -c 1 -o $O/c5s2 python bench.py --config c5 --frames 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5s2.log 2>&1
summ c5s2
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows" -c 1 -o $O/c4s2 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4s2.log 2>&1
summ c4s2
