# round-2 checkpoint: every GPU test, the full bench + reference arm, the ncu launch list of
# one step (-> traffic json), ncu --set full of the top kernels; $1 = tag
T=${1:-r2}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_l.log 2>&1
python tools/make_traffic.py gpurun_out/${T}_launches.csv gpurun_out/${T}_ncu_traffic.json > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_rag|k_resolve|k_relax_first|k_levels|k_jump|k_relabel_seg|k_grad_s2" -c 7 -o gpurun_out/${T}_top $B > gpurun_out/${T}_top.log 2>&1
python - "$T" <<'PY'
import json, sys
T = sys.argv[1]
for l in open('gpurun_out/%s_bench.log' % T):
    if l.startswith('{'):
        d = json.loads(l)
        print('value', round(d['value']), 'ms', round(d['ms_per_step'], 3), 'dom', d['roofline']['kernel'], round(d['roofline']['frac'], 4))
        print(json.dumps({k: round(v, 3) for k, v in d['phases_ms_per_step'].items()}))
        print('e2e', d.get('e2e'))
        print('grad', d.get('gradient_prepass'))
        print({k: (v.get('step_ms_min'), v.get('hbm_frac')) for k, v in (d.get('other_configs') or {}).items()})
PY
tail -c 300 gpurun_out/${T}_ref.log
