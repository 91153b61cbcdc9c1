# sync-free small-input ws_segment: parity (segment tests in both modes), then C1 / C5 timing A/B
timeout 900 python -m pytest tests -m gpu -x -q -k "segment or smoke" > gpurun_out/sm_t1.log 2>&1; echo "small rc=$?"; tail -1 gpurun_out/sm_t1.log
WS_NO_SMALL=1 timeout 900 python -m pytest tests -m gpu -x -q -k "segment" > gpurun_out/sm_t0.log 2>&1; echo "regular rc=$?"; tail -1 gpurun_out/sm_t0.log
bash tools/ab_small.sh WS_NO_SMALL
