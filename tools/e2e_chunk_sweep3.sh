#!/bin/bash
# e2e chunking for c3 / c4 / c1, two alternating repetitions
O=gpurun_out
for rep in 1 2; do
  for c in c3 c4; do
    for spec in "64 4" "64 1" "128 1" "32 1" "16 1"; do
      set -- $spec
      python bench.py --config $c --no-cpu-baseline --e2e-chunk $1 --e2e-tail $2 --steps 20 --warmup 5 \
        > $O/e2ee_${c}_$1_$2_$rep.json 2> $O/e2ee_${c}_$1_$2_$rep.err
      python - $c $1 $2 $rep <<'PY'
import json, sys
n, c, t, r = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/e2ee_{n}_{c}_{t}_{r}.json").read().strip().splitlines()[-1])
    e = d["e2e"]
    print(f"rep {r} {n} chunk {c} tail {t}: e2e {e['ms_per_step']:.4f} ms  chunks {e['chunk_frames']}")
except Exception as ex:
    print(n, c, t, "ERR", ex)
PY
    done
  done
done
