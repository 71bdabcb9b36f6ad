#!/bin/bash
# ncu --set full with source of the c5 level-0 plane kernel (16-frame chunk, 8K, N_b = 18)
O=gpurun_out
HOGB200_TUNE=0 ncu --set full --import-source on --clock-control none -k regex:k_planes -c 1 \
  -o $O/c5_planes_full python bench.py --config c5 --frames 16 --steps 1 --warmup 0 --no-e2e \
  --no-cpu-baseline > $O/c5_planes_full.log 2>&1
ncu -i $O/c5_planes_full.ncu-rep --page source --csv --print-source sass > $O/c5_planes_sass.csv 2>/dev/null
python tools/ncu_summary.py $O/c5_planes_full.ncu-rep 25 > $O/c5_planes_summary.txt 2>&1
rm -f $O/c5_planes_full.ncu-rep
