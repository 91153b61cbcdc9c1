B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv $B > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rag|k_levels|k_dense|k_levelmap" -c 4 -o gpurun_out/prof_v5a $B > gpurun_out/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_edges|k_flatten|k_hook" -c 3 -o gpurun_out/prof_v5b $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_relax_first|k_resolve|k_jump|k_union" -c 4 -o gpurun_out/prof_v5c $B > gpurun_out/ncu_c.log 2>&1
ls -la gpurun_out
