# A/B of an env-gated variant: bench phases without and with "$1"
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export $1=${2:-1}; else unset $1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/ab_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$1=$v', round(d['ms_per_step'],2), {k: round(x,2) for k,x in p.items()})
"
done
