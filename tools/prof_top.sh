# ncu --set full of each top kernel of one C4 bench step (one launch each); $1 = tag
T=${1:-top}
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
for k in k_rag k_resolve k_relax_first k_jumpv k_levels k_relabel_seg k_grad_s2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(void )?(ws::)?$k" -c 1 -o gpurun_out/${T}_$k $B > gpurun_out/${T}_$k.log 2>&1
  tail -1 gpurun_out/${T}_$k.log
done
