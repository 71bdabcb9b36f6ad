#!/bin/bash
# k_grad_bin sub-bands per plane band (HOGB200_SUBBANDS) for the small-batch regimes:
# the 64-frame shard of an 8-GPU c2 run and the single c1 frame.
O=gpurun_out
for S in 0 1 2 4 5 8; do
  HOGB200_SUBBANDS=$S python bench.py --shard-of 8 --no-cpu-baseline --no-e2e --steps 30 > $O/sb_shard8_$S.json 2>/dev/null
  HOGB200_SUBBANDS=$S python bench.py --config c1 --no-cpu-baseline --no-e2e --steps 30 > $O/sb_c1_$S.json 2>/dev/null
done
python - <<'PY'
import json
for tag in ("shard8", "c1"):
    for S in (0, 1, 2, 4, 5, 8):
        try:
            d = json.loads(open(f"gpurun_out/sb_{tag}_{S}.json").read().strip().splitlines()[-1])
            dg = d["diagnostics"]
            print(tag, "S1", S or "auto", f"{d['ms_per_step']:.4f} ms", dg["band_rows"]["used"],
                  {k: round(v, 4) for k, v in dg["stages_ms_diagnostic"].items()})
        except Exception as e:
            print(tag, S, "ERR", e)
PY
