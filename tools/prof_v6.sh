B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol"
ncu --set full --clock-control none --import-source on -k regex:"k_levels|k_jump|k_union|k_relabel|k_root_merge|k_dense" -c 6 -o gpurun_out/prof_v6a $B > gpurun_out/ncu_6a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_edges|k_relax_round|k_hook|k_levelmap" -c 4 -o gpurun_out/prof_v6b $B > gpurun_out/ncu_6b.log 2>&1
