B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"k_relax_first|k_resolve|k_jump|k_union|k_rag|k_levels" -c 6 -o gpurun_out/prof_v3a $B > gpurun_out/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_relax_round" -c 1 -o gpurun_out/prof_v3b $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_edge_min" -c 1 -o gpurun_out/prof_v3c $B > gpurun_out/ncu_c.log 2>&1
ls -la gpurun_out
