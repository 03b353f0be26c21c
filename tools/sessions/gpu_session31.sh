timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fp32 or mat32 or materialised or determinism or fused" > gpurun_out/pytest_s31.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_s31.log
timeout 600 python tools/bench_configs.py 3 4 5 > gpurun_out/bc31.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/bc31.jsonl'):
    d=json.loads(l); print(d['cfg'], d['fused_fp32']['ms'], d['materialised']['write_ms'])"
