# ncu launch lists of one ws_segment call of C1 and C5 (graph replay and, with WS_NO_SMALL=1, the regular path)
for c in C1 C5; do
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sl_$c.csv python tools/small_prof.py $c > gpurun_out/sl_$c.log 2>&1
WS_NO_SMALL=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slr_$c.csv python tools/small_prof.py $c > gpurun_out/slr_$c.log 2>&1
done
python tools/small_bench.py C1 C5
WS_NO_SMALL=1 TAG=regular python tools/small_bench.py C1 C5
