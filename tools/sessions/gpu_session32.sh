mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_final.json 2>gpurun_out/bench_ref_final.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py 1 3 4 5 > gpurun_out/bench_configs_final.jsonl 2>&1; echo "cfgs rc=$?"
timeout 1500 python tools/bench_configs.py full > gpurun_out/full_size_final.jsonl 2>&1; echo "full rc=$?"
timeout 900 python tools/paper_figures.py > gpurun_out/paper_figures_final.jsonl 2>&1; echo "figs rc=$?"
timeout 900 python tools/bench_app_a.py > gpurun_out/bench_app_a_final.jsonl 2>&1; echo "appa rc=$?"
