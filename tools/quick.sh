# quick GPU iteration: parity tests + a short bench (no e2e / cpu baseline)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -3 gpurun_out/q_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs $BENCH_ARGS > gpurun_out/q_bench.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/q_bench.log'):
    if l.startswith('{'):
        d = json.loads(l)
        print('value', round(d['value']), 'ms', round(d['ms_per_step'], 3))
        print(json.dumps({k: round(v, 3) for k, v in d['phases_ms_per_step'].items()}))
        print(d.get('input_stats'))
PY
tail -2 gpurun_out/q_bench.log | cut -c1-300
