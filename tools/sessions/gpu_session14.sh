mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s14.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_s14.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s14.json 2>gpurun_out/bench_s14.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_s14.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'], d['gpu_launches'])"
