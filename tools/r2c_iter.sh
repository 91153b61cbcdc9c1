# round 2 iteration: $1 = tag; GPU suite (minus the slow full-size oracle file), quick C4 bench; optional A/B env in $2
T=${1:-it}
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_fullsize_oracle_gpu.py > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
bash tools/quick_bench.sh ${T}
if [ -n "$2" ]; then bash tools/ab.sh $2; fi
