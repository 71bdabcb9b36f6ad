# bench lines for every config + the reference arm (gpurun_out/final_*)
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.txt 2>&1
for c in c2 c1 c3 c4; do python bench.py --config $c > $O/final_bench_$c.json 2> $O/final_bench_$c.err; done
python bench.py --config c5 --steps 3 --warmup 3 > $O/final_bench_c5.json 2> $O/final_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/final_bench_ref_c2.json 2>&1
