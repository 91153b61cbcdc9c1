# ncu --set full of the kernels matching $1 (count $2) in one bench step; report under gpurun_out/$3
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} -o gpurun_out/$3 $B > gpurun_out/$3.log 2>&1
tail -3 gpurun_out/$3.log
