# short C4 bench (no e2e / cpu baseline / context lines); $1 = tag
T=${1:-qb}
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs $BENCH_ARGS > gpurun_out/${T}_bench.log 2>&1
python - "$T" <<'PY'
import json, sys
for l in open('gpurun_out/%s_bench.log' % sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print('value', round(d['value']), 'ms', round(d['ms_per_step'], 3))
        print(json.dumps({k: round(v, 3) for k, v in d['phases_ms_per_step'].items()}))
PY
tail -2 gpurun_out/${T}_bench.log | cut -c1-300
