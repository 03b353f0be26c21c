timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s26.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_s26.log
timeout 600 python tools/bench_configs.py 4 5 > gpurun_out/bc26.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/bc26.jsonl'):
    d=json.loads(l); print(d['cfg'], d['fused_fp64']['ms'], d['fused_fp64']['fp64_frac_of_nominal'])"
