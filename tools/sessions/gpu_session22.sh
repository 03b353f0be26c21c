timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fp64 or sweep or determinism" > gpurun_out/pytest_s22.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_s22.log
timeout 600 python tools/bench_configs.py 4 5 > gpurun_out/bench_configs_s22.jsonl 2>&1; echo "cfgs rc=$?"; python -c "
import json
for l in open('gpurun_out/bench_configs_s22.jsonl'):
    d=json.loads(l); print(d['cfg'], d['fused_fp64'])"
