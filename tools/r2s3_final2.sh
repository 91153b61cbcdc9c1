# session-3 final: full GPU suite, full bench + reference arm, ncu launch list (-> traffic json),
# ncu --set full of each top kernel; $1 = tag
T=${1:-r02s3c}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_l.log 2>&1
python tools/make_traffic.py gpurun_out/${T}_launches.csv gpurun_out/${T}_ncu_traffic.json > /dev/null 2>&1
bash tools/prof_top.sh ${T}
grep '^{' gpurun_out/${T}_bench.log | tail -1 | cut -c1-400
