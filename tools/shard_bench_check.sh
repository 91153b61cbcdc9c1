# library sharded path: tests, then the contract launch `bench.py --gpus 2` (re-exec under
# torchrun; WS_BENCH_SHARE_GPU=1: both ranks on the one GPU over gloo) vs the unsharded run
timeout 900 python -m pytest tests/test_shard_lib_gpu.py tests/test_shard_gpu.py -x -q > gpurun_out/shlib.log 2>&1; echo rc=$? >> gpurun_out/shlib.log; tail -2 gpurun_out/shlib.log
A="--shape 64,512,512 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-paper-protocol --no-other-configs"
WS_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 $A > gpurun_out/sb_2.log 2>&1
timeout 600 python bench.py $A > gpurun_out/sb_1.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/sb_1.log", "gpurun_out/sb_2.log"):
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(f, "n_gpus", d["n_gpus"], "counts", d["input_stats"]["level_counts"], d["config"].get("transport"))
PY
tail -3 gpurun_out/sb_2.log | cut -c1-300
