timeout 900 python -m pytest tests -m gpu -x -q -k "segment or smoke or determinism" > gpurun_out/sm_t1.log 2>&1; echo "graph rc=$?"; tail -1 gpurun_out/sm_t1.log
bash tools/ab_small.sh WS_NO_GRAPH
