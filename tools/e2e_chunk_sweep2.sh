#!/bin/bash
# e2e chunking, repeated alternating runs (c2 whole batch and the 64-frame shard)
O=gpurun_out
for rep in 1 2 3; do
  for n in 0 8; do
    for spec in "64 4" "64 1" "128 1" "256 1"; do
      set -- $spec
      python bench.py --config c2 --shard-of $n --no-cpu-baseline --e2e-chunk $1 --e2e-tail $2 --steps 20 --warmup 5 \
        > $O/e2ed_${n}_$1_$2_$rep.json 2> $O/e2ed_${n}_$1_$2_$rep.err
      python - $n $1 $2 $rep <<'PY'
import json, sys
n, c, t, r = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/e2ed_{n}_{c}_{t}_{r}.json").read().strip().splitlines()[-1])
    e = d["e2e"]
    print(f"rep {r} shard-of {n} chunk {c} tail {t}: e2e {e['ms_per_step']:.4f} ms  chunks {e['chunk_frames']}")
except Exception as ex:
    print(n, c, t, "ERR", ex)
PY
    done
  done
done
