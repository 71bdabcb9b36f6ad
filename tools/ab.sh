for t in 1 0; do
  HOGB200_TMA=$t timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_$t.json'));print('TMA=$t', round(d['ms_per_step'],4), d['config']['stages_ms_diagnostic'], round(d['roofline']['frac'],3))"
done
