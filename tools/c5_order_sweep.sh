#!/bin/bash
# c5 pyramid: level -> stream assignment and issue order within a chunk
O=gpurun_out
for as in rr lpt; do
  for od in asc desc asc-desc; do
    HOGB200_PYR_ASSIGN=$as HOGB200_PYR_ORDER=$od python bench.py --config c5 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline \
      > $O/c5o_${as}_${od}.json 2> $O/c5o_${as}_${od}.err
  done
done
python - <<'PY'
import json
for a in ("rr", "lpt"):
    for o in ("asc", "desc", "asc-desc"):
        try:
            d = json.loads(open(f"gpurun_out/c5o_{a}_{o}.json").read().strip().splitlines()[-1])
            print("assign", a, "order", o, f"{d['ms_per_step']:.2f} ms")
        except Exception as e:
            print(a, o, "ERR", e)
PY
