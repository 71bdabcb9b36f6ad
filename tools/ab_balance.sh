O=gpurun_out
for bal in 0 1; do
  for c in c3 c2 c4; do
    HOGB200_BALANCE_STRIPS=$bal python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 > $O/abl.json 2>&1
    python -c "import json;d=json.loads(open('$O/abl.json').read().strip().splitlines()[-1]);print('bal=$bal $c', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['config']['band_rows']['used'], {k:round(v,4) for k,v in d['config']['stages_ms_diagnostic'].items()})" || tail -3 $O/abl.json
  done
  HOGB200_BALANCE_STRIPS=$bal python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 2 --warmup 2 > $O/abl.json 2>&1
  python -c "import json;d=json.loads(open('$O/abl.json').read().strip().splitlines()[-1]);print('bal=$bal c5', round(d['ms_per_step'],3), d['config']['one_stream_diagnostic'])" || tail -3 $O/abl.json
done
