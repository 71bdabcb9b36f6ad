# Plane kernel, wide variants (NW >= 6): rows per group 2 instead of 4 (A/B on c5), and an ncu capture of c3's plane kernel.
O=gpurun_out
bash tools/ab_r2.sh paper_1703_06256_b200/libhogb200.so build/libhog_gw2.so -- c5 > $O/r2e_gw_ab.txt 2>&1
HOGB200_TUNE=0 ncu --set full --import-source on --clock-control none -k regex:k_planes -c 1 \
  -o $O/c3_planes_full python bench.py --config c3 --steps 1 --warmup 0 --no-e2e \
  --no-cpu-baseline > $O/c3_planes_full.log 2>&1
ncu -i $O/c3_planes_full.ncu-rep --page source --csv --print-source sass > $O/c3_planes_sass.csv 2>/dev/null
python tools/ncu_summary.py $O/c3_planes_full.ncu-rep 25 > $O/c3_planes_summary.txt 2>&1
rm -f $O/c3_planes_full.ncu-rep
