# Launch lists of the timed region only (NVTX range "timed" in bench.py; the
# pipelines' construction-time band-row tuning launches are excluded), plus
# one ncu --set full of the c4 plane kernel at the tuned R = 80.
O=gpurun_out
for c in c2 c4; do
  ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/tl_${c}_launches.csv python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/tl_$c.log 2>&1
done
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/tl_c5_launches.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/tl_c5.log 2>&1
HOGB200_TUNE=0 HOGB200_BAND_ROWS=80 ncu --set full --clock-control none --import-source on -k regex:"k_planes" -c 1 \
    -o $O/c4_planes_R80 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/tl_c4f.log 2>&1
ncu -i $O/c4_planes_R80.ncu-rep --page raw --csv > $O/c4_planes_R80_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/c4_planes_R80.ncu-rep 25 > $O/c4_planes_R80_summary.txt 2>&1
rm -f $O/c4_planes_R80.ncu-rep
