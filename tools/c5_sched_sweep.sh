O=gpurun_out
for ch in 16 8; do for st in 2 3 4 6; do
  python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --pyr-streams $st --pyr-chunk $ch > $O/c5s.json 2>&1
  python -c "import json;d=json.loads(open('$O/c5s.json').read().strip().splitlines()[-1]);print('chunk=$ch streams=$st', round(d['ms_per_step'],3))" || tail -2 $O/c5s.json
done; done
