for R in 0 32 64 128; do
  for c in c3 c5; do
    st=10; [ $c = c5 ] && st=2
    if [ $R = 0 ]; then unset HOGB200_BAND_ROWS; else export HOGB200_BAND_ROWS=$R; fi
    timeout 400 python bench.py --config $c --no-e2e --no-cpu-baseline --steps $st --warmup 2 > gpurun_out/r.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/r.json'));print('R=$R $c', round(d['ms_per_step'],3), (d['config'].get('stages_ms_diagnostic') or {}).get('planes_grid'), round(d['roofline']['frac'],3))"
  done
done
