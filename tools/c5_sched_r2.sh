#!/bin/bash
# c5 pyramid schedule: frames per chunk x level streams
O=gpurun_out
for ch in 8 16; do
  for s in 4 6 8; do
    python bench.py --config c5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --pyr-chunk $ch \
      --pyr-streams $s > $O/c5s_${ch}_${s}.json 2> $O/c5s_${ch}_${s}.err
  done
done
python - <<'PY'
import json
for ch in (8, 16):
    for s in (4, 6, 8):
        try:
            d = json.loads(open(f"gpurun_out/c5s_{ch}_{s}.json").read().strip().splitlines()[-1])
            print("chunk", ch, "streams", s, f"{d['ms_per_step']:.2f} ms", f"pipeline frac {d['pipeline_roofline']['frac']:.3f}")
        except Exception as e:
            print(ch, s, "ERR", e)
PY
