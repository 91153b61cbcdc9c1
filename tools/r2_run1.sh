# round 2, first GPU call: host facts, full GPU test suite (incl. full-size oracle parity), quick bench
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA -k "fullsize_oracle" > gpurun_out/r2_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fullsize.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_fullsize_oracle_gpu.py > gpurun_out/r2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs > gpurun_out/r2_bench1.log 2>&1
tail -5 gpurun_out/r2_fullsize.log; tail -3 gpurun_out/r2_pytest.log; tail -c 600 gpurun_out/r2_bench1.log
