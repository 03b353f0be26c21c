mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_app_a_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_app_a_s6.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_app_a_s6.log
timeout 600 python tools/bench_app_a.py > gpurun_out/bench_app_a_s6.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/bench_app_a_s6.jsonl | tail -8
