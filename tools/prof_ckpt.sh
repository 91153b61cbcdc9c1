# checkpoint: full bench (N=1) + launch list + ncu traffic json + full sets of the top kernels
set -x
timeout 900 python bench.py > gpurun_out/ckpt_bench.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ckpt_launches.csv $B > gpurun_out/ckpt_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rag|k_resolve|k_relax_first|k_levels|k_jump|k_edges" -c 6 -o gpurun_out/ckpt_top $B > gpurun_out/ckpt_top.log 2>&1
ls -la gpurun_out | tail -5
