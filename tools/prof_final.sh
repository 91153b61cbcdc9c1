# end-of-session artefacts: full bench (N=1, all configs), reference arm, ncu launch list of
# one step, ncu --set full of the top kernels; $1 = tag
T=${1:-final}
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_l.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_rag|k_resolve|k_relax_first|k_levels|k_jump|k_edges" -c 6 -o gpurun_out/${T}_top $B > gpurun_out/${T}_top.log 2>&1
ls -la gpurun_out | tail -8
