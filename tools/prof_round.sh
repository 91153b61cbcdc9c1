# one launch list of a full bench step + full ncu sets of the top kernels (run under gpurun)
set -x
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rag|k_levels|k_relax_first|k_resolve" -c 4 -o gpurun_out/prof_top $B > gpurun_out/ncu_top.log 2>&1
ls -la gpurun_out
