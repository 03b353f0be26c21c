for v in 2 4; do XLMIMO_MT2_SM=$v timeout 600 python tools/bench_configs.py 4 > gpurun_out/bc23_$v.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/bc23_$v.jsonl'):
    d=json.loads(l); print('$v', d['cfg'], d['fused_fp64']['ms'], d['fused_fp64']['fp64_frac_of_nominal'])"; done
XLMIMO_MT2_SM=4 timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "fp64" 2>&1 | tail -1
