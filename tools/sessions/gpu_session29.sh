timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s29.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_s29.log
timeout 1500 python tools/bench_configs.py full > gpurun_out/full_size.jsonl 2> gpurun_out/full_size.err; echo "full rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/full_size.jsonl'):
    d=json.loads(l)
    print(d['cfg'], d['drops'], {k:(round(v['ms'],2), round(v['drops_per_s'])) for k,v in d.items() if isinstance(v,dict)})
PY
timeout 600 python tools/bench_app_a.py 2>&1 | head -3 | cut -c1-200
