# compute-sanitizer memcheck / initcheck / synccheck / racecheck over tools/sanitize_run.py; $1 = output file
O=${1:-gpurun_out/sanitizers.txt}
: > $O
for t in memcheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1
  echo "$t: $(grep 'ERROR SUMMARY' gpurun_out/san_$t.log | tail -1)" >> $O
done
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 100000 python tools/sanitize_run.py > gpurun_out/san_racecheck.log 2>&1
echo "racecheck (analysis mode: every reported race, grouped by kernel and the two source lines):" >> $O
python tools/race_group.py gpurun_out/san_racecheck.log >> $O
grep "RACECHECK SUMMARY" gpurun_out/san_racecheck.log | tail -1 >> $O
grep -h " ok" gpurun_out/san_memcheck.log >> $O
cat $O
