#!/bin/bash
# round-1 re-entry check: GPU parity, smoke, bench, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s5_gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s5.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_s5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s5.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_s5.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_s5.json 2>gpurun_out/bench_s5.err; echo "bench rc=$?"
cat gpurun_out/bench_s5.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_s5.json 2>gpurun_out/bench_ref_s5.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_s5.json
timeout 600 python tools/bench_configs.py > gpurun_out/bench_configs_s5.jsonl 2>gpurun_out/bench_configs_s5.err; echo "cfgs rc=$?"; cat gpurun_out/bench_configs_s5.jsonl
