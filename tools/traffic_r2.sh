#!/bin/bash
# DRAM bytes of one k_planes launch per config (row-major planes, library band rows),
# plus one ncu --set full capture of the c2 plane kernel.  -> gpurun_out/tr2_*.csv
O=gpurun_out
for c in c2 c3 c4; do
  HOGB200_TUNE=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_planes -c 1 --csv --log-file $O/tr2_$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/tr2_$c.log 2>&1
done
HOGB200_TUNE=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:k_planes -c 1 --csv --log-file $O/tr2_c5.csv \
  python bench.py --config c5 --frames 16 --pyr-chunk 16 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/tr2_c5.log 2>&1
HOGB200_TUNE=0 ncu --set full --import-source on --clock-control none -k regex:k_planes -c 1 -o $O/tr2_c2_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/tr2_c2_full.log 2>&1
