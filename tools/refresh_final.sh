#!/bin/bash
# Round-end refresh without ncu captures: GPU tests, smoke, bench (+ reference arm), the bench
# launch list, Appendix A / large-K timings and the paper-figure workloads.
#   bash tools/refresh_final.sh OUTDIR   (under gpurun_out/, merged back by gpurun)
set -x
O=${1:-gpurun_out/final}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
      python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 python tools/bench_app_a.py > $O/bench_app_a.jsonl 2> $O/bench_app_a.err
timeout 900 python tools/paper_figures.py > $O/paper_figures.jsonl 2> $O/paper_figures.err
timeout 600 python tools/ab_mt2k.py 49,56,72,80,88,96,100,112,120,128 product > $O/mt2_k_sweep.txt 2>&1
