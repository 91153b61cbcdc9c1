# compute-sanitizer memcheck / initcheck / synccheck / racecheck over tools/sanitize_run.py; $1 = output file
O=${1:-gpurun_out/sanitizers.txt}
: > $O
for t in memcheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1
  echo "$t: $(grep 'ERROR SUMMARY' gpurun_out/san_$t.log | tail -1)" >> $O
done
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1
echo "racecheck (shared-memory hazards, grouped by source line):" >> $O
grep -o "Race reported between [A-Za-z]* access at .* in [a-z_0-9]*\.cu[h]*:[0-9]*" gpurun_out/san_racecheck.log | sed 's/(.*)//' | sort | uniq -c | sort -rn | head -20 >> $O
grep "RACECHECK SUMMARY" gpurun_out/san_racecheck.log | tail -1 >> $O
grep -h " ok" gpurun_out/san_memcheck.log >> $O
cat $O
