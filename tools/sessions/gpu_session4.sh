#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s4.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_s4.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_s4.json 2>gpurun_out/bench_s4.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_s4.json'));print(d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'], d['e2e'], d['cpu_baseline'])"
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_s4_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s4.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_s4.log 2>&1; echo "ncu rc=$?"
