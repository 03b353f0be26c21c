mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s18.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_s18.log
timeout 600 python tools/bench_configs.py 1s > gpurun_out/cfg1_steady.jsonl 2>&1; echo "cfg1s rc=$?"; cat gpurun_out/cfg1_steady.jsonl | cut -c1-700
