O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/gpu_tests7.log 2>&1
for ty in 4 5; do
  HOGB200_SCORES_TY=$ty python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/ty.json 2>&1
  python -c "import json;d=json.loads(open('$O/ty.json').read().strip().splitlines()[-1]);print('ty=$ty c4', round(d['ms_per_step'],4))" || tail -3 $O/ty.json
done
python bench.py --config c4 --no-cpu-baseline --no-e2e > $O/ty.json 2>&1
python -c "import json;d=json.loads(open('$O/ty.json').read().strip().splitlines()[-1]);print('auto c4', round(d['ms_per_step'],4))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_scores_rows -c 2 --log-file $O/ty_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
HOGB200_SCORES_TY=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_scores_rows -c 2 --log-file $O/ty4_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/ty_c5.json 2>&1
python -c "import json;d=json.loads(open('$O/ty_c5.json').read().strip().splitlines()[-1]);print('c5', round(d['ms_per_step'],3))"
