# compute-sanitizer over the engine paths (scripts/sanitize_workload.py);
# one summary line per (tool, path) into gpurun_out/r02_sanitize.txt
out=gpurun_out/r02_sanitize.txt
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  for path in dense packed worklist summary segments relabel hubs multi peer; do
    log=gpurun_out/san_${tool}_${path}.log
    timeout 400 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py $path > $log 2>&1
    rc=$?
    echo "$tool $path rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tail -1) $(grep -h 'steps bit-exact' $log | tail -1)" >> $out
  done
done
cat $out
