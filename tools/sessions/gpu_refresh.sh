#!/bin/bash
# Round-end refresh of every measured artefact (one GPU): tests, smoke, bench (+ reference
# arm), per-config paths, full sizes, cfg1 steady state, paper figures, Appendix A / large K,
# fp32 paths, the bench launch list under ncu.
mkdir -p gpurun_out
T=${1:-r}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$T.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2>gpurun_out/bench_$T.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$T.json 2>gpurun_out/bench_ref_$T.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py 1 3 4 5 > gpurun_out/bench_configs_$T.jsonl 2>&1; echo "cfgs rc=$?"
timeout 1500 python tools/bench_configs.py full > gpurun_out/full_size_$T.jsonl 2>&1; echo "full rc=$?"
timeout 600 python tools/bench_configs.py 1s > gpurun_out/cfg1_steady_$T.jsonl 2>&1; echo "1s rc=$?"
timeout 900 python tools/paper_figures.py > gpurun_out/paper_figures_$T.jsonl 2>&1; echo "figs rc=$?"
timeout 900 python tools/bench_app_a.py > gpurun_out/bench_app_a_$T.jsonl 2>&1; echo "appa rc=$?"
timeout 600 python tools/time_fused32.py > gpurun_out/fused32_$T.json 2>&1; echo "f32 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_$T.log 2>&1; echo "ncu rc=$?"
