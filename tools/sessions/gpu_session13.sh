mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s13.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_s13.log
timeout 600 python tools/bench_configs.py 3 5 > gpurun_out/bench_configs_s13.jsonl 2>&1; echo "cfgs rc=$?"; cut -c1-600 gpurun_out/bench_configs_s13.jsonl
timeout 600 python tools/bench_app_a.py > gpurun_out/bench_app_a_s13.jsonl 2>&1; echo "appa rc=$?"; tail -1 gpurun_out/bench_app_a_s13.jsonl | cut -c1-500
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s13.json 2>gpurun_out/bench_s13.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_s13.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'])"
