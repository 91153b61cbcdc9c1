# A/B of an env switch $1 on C4 (phases) and the small configs C1, C5 (ms/step)
for v in 0 1; do
  if [ $v = 1 ]; then export $1=1; else unset $1; fi
  for c in C4 C1 C5; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/abs_${c}_$v.log 2>&1
    python -c "
import json
for l in open('gpurun_out/abs_${c}_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$1=$v $c', round(d['ms_per_step'],3), 'min', round(d['step_ms']['min'],3), {k: round(x,3) for k,x in p.items() if k.startswith('watershed.relax')})
"
  done
done
