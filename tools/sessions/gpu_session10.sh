mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_large_k_gpu.py tests/test_paper_figures_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_s10.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_s10.log
timeout 600 python tools/bench_app_a.py > gpurun_out/bench_app_a_s10.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/bench_app_a_s10.jsonl | tail -3 | cut -c1-400
