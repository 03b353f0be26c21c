mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "mat32 or materialised or determinism" > gpurun_out/pytest_s20.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_s20.log
timeout 600 python tools/bench_configs.py 3 4 5 > gpurun_out/bench_configs_s20.jsonl 2>&1; echo "cfgs rc=$?"; python -c "
import json
for l in open('gpurun_out/bench_configs_s20.jsonl'):
    d=json.loads(l); m=d['materialised']; print(d['cfg'], round(m['write_ms'],3), round(m['write_gbs'],1), round(m['stream_ms'],3), round(m['stream_gbs'],1))"
