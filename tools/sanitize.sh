# compute-sanitizer over every device entry point (tools/sanitize_paths.py)
O=${1:-gpurun_out}
python tools/sanitize_paths.py > $O/sanitize_bare.txt 2>&1 || { cat $O/sanitize_bare.txt; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/sanitize_summary.txt
  tail -3 $O/sanitize_$tool.txt >> $O/sanitize_summary.txt
done
