# A/B of binning-kernel variants (HOGB200_LIB) on c2 and c4: step and grad_bin stage time
for lib in "" build/libhog_k1u2.so build/libhog_k1u4.so; do
  for c in c2 c4; do
    HOGB200_LIB=$lib timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/abb.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/abb.json'));print('${lib:-default} $c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['config']['stages_ms_diagnostic'].items()})" || tail -3 gpurun_out/abb.json
  done
done
