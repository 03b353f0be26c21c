timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s24.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_s24.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b24.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b24.json'));r=d['roofline'];print(round(d['ms_per_step'],3), round(r['launch_ms'],3), round(r['frac'],4))"
timeout 600 python tools/bench_configs.py 3 4 5 > gpurun_out/bc24.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/bc24.jsonl'):
    d=json.loads(l); print(d['cfg'], d['fused_fp64']['ms'])"
