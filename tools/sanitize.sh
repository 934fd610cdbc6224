# compute-sanitizer over the smoke test and tools/sanitize.py (every kernel family)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
out=gpurun_out/sanitizer.txt; : > $out
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool: smoke" >> $out
  timeout 900 $CS --tool $tool --print-limit 20 python __graft_entry__.py smoke >> $out 2>&1; echo "rc=$?" >> $out
  echo "=== $tool: tools/sanitize.py" >> $out
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize.py >> $out 2>&1; echo "rc=$?" >> $out
done
grep -E "^===|ERROR SUMMARY|rc=|ok" $out
