# A/B of prebuilt abso/lib_*.so variants (copied over libws_b200.so): short C4 bench, all phases; $1 = reps
for rep in $(seq ${1:-2}); do
for f in abso/lib_*.so; do
  cp "$f" paper_2410_08946_b200/libws_b200.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs $BENCH_ARGS > gpurun_out/abso.log 2>&1
  python -c "
import json
for l in open('gpurun_out/abso.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['phases_ms_per_step']; print('$f', round(d['ms_per_step'],2), {k: round(x,2) for k,x in p.items()})
"
done
done
