# Round-1 (second pass) evidence for c3/c4/c5; ncu reports are summarised on
# the box (raw CSV + tools/ncu_summary.py) and deleted: gpurun_out/ must stay < 64 MiB.
set -x
O=gpurun_out
summ() {  # report -> text summary + raw csv, then drop the report
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/$1.ncu-rep 25 > $O/$1_summary.txt 2>&1
  rm -f $O/$1.ncu-rep
}
python -m pytest tests/test_gpu_pyramid.py -x -q > $O/pyr_tests.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/probe_cvt tools/probe_cvt.cu && build/probe_cvt > $O/probe_cvt.txt 2>&1
python bench.py --config c3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
for s in 1 2 3; do
  python bench.py --config c5 --steps 2 --warmup 2 --pyr-streams $s $([ $s != 1 ] && echo --no-cpu-baseline) > $O/bench_c5_s$s.json 2> $O/bench_c5_s$s.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c5_launches.csv python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5l.log 2>&1
for c in c3 c4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_planes -c 1 --log-file $O/${c}_traffic.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_${c}t.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_planes -c 1 --log-file $O/c5_traffic.csv python bench.py --config c5 --frames 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5t.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows|k_grad_bin" -c 2 -o $O/c4_full python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c4f.log 2>&1
summ c4_full
ncu --set full --clock-control none --import-source on -k regex:"k_scores_rows|k_resize" -c 2 -o $O/c5_full python bench.py --config c5 --frames 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5f.log 2>&1
summ c5_full
du -sh $O; ls -la $O
