O=gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined or chunked or lattice" > $O/gpu_tests6.log 2>&1
for pp in 0 1; do for c in c4 c1; do
  python bench.py --config $c --no-cpu-baseline --no-e2e --pipelined $pp > $O/pp.json 2>&1
  python -c "import json;d=json.loads(open('$O/pp.json').read().strip().splitlines()[-1]);print('pipelined=$pp $c', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['pipeline_roofline']['frac'],3))" || tail -3 $O/pp.json
done; done
