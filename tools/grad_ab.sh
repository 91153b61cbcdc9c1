# gradient v2 vs v1 (WS_GRAD_V1=1): parity tests of both, then C4 pre-pass timing
timeout 900 python -m pytest tests -m gpu -x -q -k "gradient or u16 or fullsize_gpu" > gpurun_out/ga_v2.log 2>&1; echo "v2 rc=$?"; tail -1 gpurun_out/ga_v2.log
WS_GRAD_V1=1 timeout 900 python -m pytest tests -m gpu -x -q -k "gradient" > gpurun_out/ga_v1.log 2>&1; echo "v1 rc=$?"; tail -1 gpurun_out/ga_v1.log
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export WS_GRAD_V1=1; else unset WS_GRAD_V1; fi
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/ga_b$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ga_b$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print('WS_GRAD_V1=$v gradient ms', round(d['gradient_prepass']['ms'],3), 'step', round(d['ms_per_step'],2), 'regions', d['input_stats']['regions'])
"
done
