#!/bin/bash
# A/B/... of library builds (and env switches) on the same box: alternating
# bench runs per config.
# usage: tools/ab_r2.sh "<lib>[@VAR=val,...]" "<lib>[@...]" ... -- <configs...>
# results -> gpurun_out/ab_<config>_<variant index>_<rep>.json, summary on stdout
O=gpurun_out
V=()
while [ "$1" != "--" ]; do V+=("$1"); shift; done
shift
# a config may carry extra bench args after a colon: c2:--shard-of=8
for spec_c in "$@"; do
  c=${spec_c%%:*}; xargs_=""
  [[ "$spec_c" == *:* ]] && xargs_=$(echo "${spec_c#*:}" | tr ',' ' ')
  tagc=$(echo "$spec_c" | tr ':=,' '___')
  for rep in 1 2; do
    for i in "${!V[@]}"; do
      spec=${V[$i]}; lib=${spec%%@*}; envs=""
      [[ "$spec" == *@* ]] && envs=$(echo "${spec#*@}" | tr ',' ' ')
      env HOGB200_LIB=$lib $envs python bench.py --config $c $xargs_ --steps 20 --warmup 5 --no-e2e \
        --no-cpu-baseline > $O/ab_${tagc}_${i}_${rep}.json 2> $O/ab_${tagc}_${i}_${rep}.err
    done
  done
done
python - "${#V[@]}" "${V[@]}" -- "$@" <<'PY'
import json, sys, glob
n = int(sys.argv[1]); specs = sys.argv[2:2 + n]
cfgs = [c.replace(":", "_").replace("=", "_").replace(",", "_") for c in sys.argv[3 + n:]]
for c in cfgs:
    for i, spec in enumerate(specs):
        for f in sorted(glob.glob(f"gpurun_out/ab_{c}_{i}_*.json")):
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1])
                dg = d.get("diagnostics", {})
                print(c, i, spec, f"{d['ms_per_step']:.4f} ms", f"frac {d['roofline']['frac']:.3f}",
                      {k: round(v, 4) for k, v in dg.get("stages_ms_diagnostic", {}).items()})
            except Exception as e:
                print(c, i, spec, "ERR", e, open(f.replace('.json', '.err')).read()[-300:])
PY
