#!/bin/bash
# Refresh after an fp64-generator change: GPU tests, smoke, the fp64 kernels' ncu digests,
# their DRAM traffic, bench (+ reference arm) and the bench launch list.
#   bash tools/refresh_fp64.sh OUTDIR   (under gpurun_out/, merged back by gpurun)
set -x
O=${1:-gpurun_out/refresh}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
cap() { # tag cfg prec drops regex
  python tools/prof_gram.py $2 $3 $4 > $O/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$5 -s 1 -c 1 -o $O/$1 -f \
      python tools/prof_gram.py $2 $3 $4 > $O/ncu_$1.log 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/ncu_full_$1.txt 2>&1
  python tools/ncu_hot.py $O/$1.ncu-rep 40 > $O/ncu_hot_$1.txt 2>&1
  python tools/ncu_lines.py $O/$1.ncu-rep 40 > $O/ncu_lines_$1.txt 2>&1
}
cap mt2_cfg5_d1000 5 fp64 1000 gram_mt2
cap mt2_cfg4 4 fp64 1000 gram_mt2
cap warp_cfg1 1 fp64 1000000 gram_warp
cap mma_cfg3 3 fp64 10000 gram_mma_kernel
cp profiles/r02/ncu_traffic_bench.json $O/ncu_traffic_bench.json
python tools/ncu_traffic.py --merge $O/ncu_traffic_bench.json \
  $O/mt2_cfg5_d1000.ncu-rep:gram_fused_dmma_tiled_fp64:"cfg5 fp64 D=1000":1000 > $O/traffic.log 2>&1
rm -f $O/*.ncu-rep
cp $O/ncu_traffic_bench.json profiles/r02/ncu_traffic_bench.json  # the box's copy: bench reads it
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
      python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > $O/ncu_launch.log 2>&1
