O=gpurun_out
for lib in "" build/libhog_smemcnt.so; do
  for c in c3 c2 c4; do
    HOGB200_LIB=$lib python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 > $O/abs.json 2>&1
    python -c "import json;d=json.loads(open('$O/abs.json').read().strip().splitlines()[-1]);print('${lib:-default} $c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['config']['stages_ms_diagnostic'].items()})" || tail -3 $O/abs.json
  done
  HOGB200_LIB=$lib python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 2 --warmup 2 > $O/abs.json 2>&1
  python -c "import json;d=json.loads(open('$O/abs.json').read().strip().splitlines()[-1]);print('${lib:-default} c5', round(d['ms_per_step'],3), d['config']['one_stream_diagnostic']['step_ms'])" || tail -3 $O/abs.json
done
