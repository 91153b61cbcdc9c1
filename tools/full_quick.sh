# all GPU tests except the slow full-size oracle file, then a short bench; $1 = tag
T=${1:-fq}
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_fullsize_oracle_gpu.py > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
bash tools/quick_bench.sh $T
python -c "
import json
for l in open('gpurun_out/${T}_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('stats', {k: d['input_stats'].get(k) for k in ('regions','edges','rag_records','rag_global_emits')})
" 2>/dev/null
