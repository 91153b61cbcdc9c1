# session-3 checkpoint: full GPU suite, full bench + reference arm, ncu launch list (-> traffic
# json), ncu --set full of the top kernels, sanitizers; $1 = tag
T=${1:-r02s3}
bash tools/r2_full.sh $T
bash tools/sanitize_all.sh gpurun_out/${T}_sanitizers.txt > /dev/null 2>&1
head -8 gpurun_out/${T}_sanitizers.txt
