# one GPU iteration: tests, benches of the changed paths, e2e sweep, scores-kernel ncu
set -x
O=gpurun_out
summ() {
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/$1.ncu-rep 25 > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
python bench.py --config c4 --no-cpu-baseline > $O/it_c4.json 2> $O/it_c4.err
python bench.py --config c1 --no-cpu-baseline > $O/it_c1.json 2> $O/it_c1.err
python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > $O/it_c5.json 2> $O/it_c5.err
python tools/pcie_probe.py > $O/pcie.txt 2>&1
for a in "32 4 4" "32 6 4" "128 2 4" "64 6 8" "64 4 1"; do set -- $a
  python bench.py --steps 10 --no-cpu-baseline --e2e-chunk $1 --e2e-slots $2 --e2e-tail $3 > $O/e2e_$1_$2_$3.json 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows" -c 1 -o $O/c5s python bench.py --config c5 --frames 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5s.log 2>&1
summ c5s
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows" -c 1 -o $O/c4s python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4s.log 2>&1
summ c4s
du -sh $O
