# quick C4 bench phases under several env settings (each "A=1,B=1" or "-" for none), twice each
for rep in 1 2; do
for cfg in "$@"; do
  ( if [ "$cfg" != "-" ]; then for kv in ${cfg//,/ }; do export $kv; done; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/ab3.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab3.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$cfg', round(d['ms_per_step'],2), {k: round(x,2) for k,x in p.items()})
" )
done
done
