O=gpurun_out
python tools/e2e_timeline.py > $O/tl_new_64_4_4.txt 2>&1
python tools/e2e_timeline.py --chunk 32 --slots 3 --tail 2 > $O/tl_new_32_3_2.txt 2>&1
for a in "64 4 4" "64 2 4" "32 3 2" "32 4 4" "16 4 1" "128 2 8"; do set -- $a
  python bench.py --steps 10 --no-cpu-baseline --e2e-chunk $1 --e2e-slots $2 --e2e-tail $3 > $O/e2eN_$1_$2_$3.json 2>&1
done
python bench.py --config c4 --steps 10 --no-cpu-baseline > $O/e2eN_c4.json 2>&1
python bench.py --config c3 --steps 10 --no-cpu-baseline > $O/e2eN_c3.json 2>&1
