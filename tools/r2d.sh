# parity suite + C4 quick bench + small-config step times
T=${1:-it}
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_fullsize_oracle_gpu.py > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
bash tools/quick_bench.sh ${T}
python tools/small_bench.py C1 C5 C3 C2
