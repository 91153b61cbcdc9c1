# ncu launch list (device time + DRAM bytes per launch) of one bench step; $1 = output tag
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/$1.csv $B > gpurun_out/$1.log 2>&1
python tools/launches.py gpurun_out/$1.csv | head -40
