#!/bin/bash
# A/B the default library against variants on given configs:
#   tools/ab_lib.sh "c2 c3" build/libhog_x.so [...]
cfgs=$1; shift
for lib in default "$@"; do
  for c in $cfgs; do
    if [ "$lib" = default ]; then unset HOGB200_LIB; else export HOGB200_LIB=$PWD/$lib; fi
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "$lib $c FAILED"; tail -3 gpurun_out/ab.err; continue; }
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib', '$c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in (d['config'].get('stages_ms_diagnostic') or {}).items()}, round(d['roofline']['frac'],3))"
  done
done
