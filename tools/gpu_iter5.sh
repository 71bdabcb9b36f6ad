O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/gpu_tests5.log 2>&1
for nd in 1 2; do for c in c2 c4 c3; do
  HOGB200_K1_ND=$nd python bench.py --config $c --no-cpu-baseline --no-e2e > $O/nd.json 2>&1
  python -c "import json;d=json.loads(open('$O/nd.json').read().strip().splitlines()[-1]);print('nd=$nd $c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['config']['stages_ms_diagnostic'].items()})" || tail -3 $O/nd.json
done; done
python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/nd_c5.json 2>&1
python -c "import json;d=json.loads(open('$O/nd_c5.json').read().strip().splitlines()[-1]);print('c5', round(d['ms_per_step'],3), d['config']['one_stream_diagnostic'])"
