# round 2 GPU iteration: $1 = tag; parity tests, full bench, ncu launch list -> ncu_traffic.json
T=${1:-r2}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_l.log 2>&1
python tools/make_traffic.py gpurun_out/${T}_launches.csv gpurun_out/${T}_ncu_traffic.json > /dev/null 2>&1
python - <<PY
import json
for l in open('gpurun_out/${T}_bench.log'):
    if l.startswith('{'):
        d = json.loads(l)
        print('value', round(d['value']), 'ms', round(d['ms_per_step'], 3), 'dom', d['roofline']['kernel'], round(d['roofline']['frac'],4))
        print(json.dumps({k: round(v, 3) for k, v in d['phases_ms_per_step'].items()}))
        print('e2e', d.get('e2e'))
PY
tail -c 400 gpurun_out/${T}_bench.log
