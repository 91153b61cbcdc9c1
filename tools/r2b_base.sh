# round 2 re-entry baseline: quick C4 bench at HEAD, then the GPU suite (minus the slow full-size oracle file)
bash tools/quick_bench.sh base
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_fullsize_oracle_gpu.py > gpurun_out/base_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/base_pytest.log
tail -3 gpurun_out/base_pytest.log
