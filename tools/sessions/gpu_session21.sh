mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s21.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_s21.log
timeout 900 python tools/bench_configs.py 1 3 4 5 > gpurun_out/bench_configs_s21.jsonl 2>&1; echo "cfgs rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_s21.json 2>gpurun_out/bench_s21.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_s21.json'));print(d['value'], d['ms_per_step'], d['roofline'], d['e2e'], d['cpu_baseline']['value'])"
