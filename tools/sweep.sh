# sweep an env knob: $1 = name, rest = values; prints the step and phase times per value
name=$1; shift
for v in "$@"; do
  export $name=$v
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/sw_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/sw_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$name=$v', round(d['ms_per_step'],2), {k: round(x,2) for k,x in p.items() if x > 0.5})
"
done
