# segment-path iteration: segment parity (small + full size) and a short bench
timeout 900 python -m pytest tests -m gpu -x -q -k "segment" > gpurun_out/sq_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sq_pytest.log
tail -3 gpurun_out/sq_pytest.log
bash tools/quick_bench.sh sq
