#!/bin/bash
# First GPU session: microbenchmarks, GPU parity tests, smoke, a short bench.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 120 ./tools/peaks > gpurun_out/peaks.json 2>&1; echo "peaks rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-sample-seconds 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/peaks.json gpurun_out/bench.json
