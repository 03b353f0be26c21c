mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_app_a_gpu.py tests/test_large_k_gpu.py tests/test_paper_figures_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_s8.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_s8.log
timeout 600 python tools/bench_app_a.py > gpurun_out/bench_app_a_s8.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/bench_app_a_s8.jsonl | tail -3
