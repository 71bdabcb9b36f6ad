#!/bin/bash
# e2e copy/compute chunking for small shards (the per-GPU work of 2/4/8-GPU runs of c2)
O=gpurun_out
for n in 8 4 0; do
  for spec in "64 4" "64 1" "64 2" "32 1" "128 1" "128 2"; do
    set -- $spec
    python bench.py --config c2 --shard-of $n --no-cpu-baseline --e2e-chunk $1 --e2e-tail $2 --steps 20 --warmup 5 \
      > $O/e2ec_${n}_$1_$2.json 2> $O/e2ec_${n}_$1_$2.err
    python - $n $1 $2 <<'PY'
import json, sys
n, c, t = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/e2ec_{n}_{c}_{t}.json").read().strip().splitlines()[-1])
    e = d["e2e"]
    print(f"shard-of {n} chunk {c} tail {t}: e2e {e['ms_per_step']:.4f} ms  chunks {e['chunk_frames']}")
except Exception as ex:
    print(n, c, t, "ERR", ex)
PY
  done
done
