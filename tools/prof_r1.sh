# ncu captures for round 1 (session 2): launch list with DRAM bytes + full sets of the top kernels
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s2_launches.csv $B > gpurun_out/r1s2_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_relax_first|k_resolve|k_jump|k_relabel|k_dense|k_rag|k_levels|k_root_merge" -c 8 -o gpurun_out/r1s2_a $B > gpurun_out/r1s2_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_edges|k_relax_round|k_hook|k_flatten|k_levelmap" -c 5 -o gpurun_out/r1s2_b $B > gpurun_out/r1s2_b.log 2>&1
ls -la gpurun_out
