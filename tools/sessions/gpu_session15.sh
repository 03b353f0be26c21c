mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fp32 or determinism or fused or sweep" > gpurun_out/pytest_gpu_s15.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_s15.log
timeout 600 python tools/bench_configs.py 3 4 5 > gpurun_out/bench_configs_s15.jsonl 2>&1; echo "cfgs rc=$?"; python -c "
import json
for l in open('gpurun_out/bench_configs_s15.jsonl'):
    d=json.loads(l); print(d['cfg'], d['fused_fp32'])"
