#!/bin/bash
# usage: tools/gpu_tune2.sh <tag> "<env1>;<env2>;..." [ncu regex] [ncu env]
mkdir -p gpurun_out
TAG=$1; IFS=';' read -ra ENVS <<< "$2"; RX=${3:-}; NENV=${4:-}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_$TAG.log
i=0
for e in "${ENVS[@]}"; do
  env $e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2>gpurun_out/bench_${TAG}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$i.json'));r=d['roofline'];print('$e', round(d['ms_per_step'],3), r['kernel'], round(r['launch_ms'],3), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/bench_${TAG}_$i.err
  i=$((i+1))
done
if [ -n "$RX" ]; then env $NENV bash tools/ncu_gram.sh $TAG 2000 $RX; fi
