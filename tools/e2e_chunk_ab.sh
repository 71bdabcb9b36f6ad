#!/bin/bash
# c2 e2e: the old chunking (64-frame chunks, last one split in four) against the default
# (four chunks per step), alternating, three repetitions
O=gpurun_out
for rep in 1 2 3; do
  for spec in "64 4" "0 1"; do
    set -- $spec
    python bench.py --config c2 --no-cpu-baseline --e2e-chunk $1 --e2e-tail $2 > $O/e2ef_$1_$2_$rep.json 2> $O/e2ef_$1_$2_$rep.err
    python - $1 $2 $rep <<'PY'
import json, sys
c, t, r = sys.argv[1:]
d = json.loads(open(f"gpurun_out/e2ef_{c}_{t}_{r}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(f"rep {r} chunk {c} tail {t}: e2e {e['ms_per_step']:.4f} ms  chunks {e['chunk_frames']}  device step {d['ms_per_step']:.4f} ms")
PY
  done
done
