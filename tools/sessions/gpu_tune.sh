#!/bin/bash
# usage: tools/gpu_tune.sh "<cfg list>" <tag> [ncu regex]
mkdir -p gpurun_out
CFGS=${1:-"0"}; TAG=${2:-t}; RX=${3:-}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_$TAG.log
for c in $CFGS; do
  XLMIMO_SPLIT_CFG=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg$c.json 2>gpurun_out/bench_${TAG}_cfg$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_cfg$c.json'));r=d['roofline'];print('cfg $c', round(d['ms_per_step'],3), r['kernel'], round(r['launch_ms'],3), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/bench_${TAG}_cfg$c.err
done
if [ -n "$RX" ]; then bash tools/ncu_gram.sh $TAG 2000 $RX; fi
