#!/bin/bash
# ncu capture of the fused Gram kernel (one launch) + launch list of one bench step.
# usage: tools/ncu_gram.sh <tag> [n_drops] [regex]
TAG=${1:-r1}; D=${2:-2000}; RX=${3:-gram_small}
mkdir -p gpurun_out
python tools/prof_sweep.py $D > gpurun_out/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$RX -s 1 -c 1 \
    -o gpurun_out/gram_$TAG -f python tools/prof_sweep.py $D > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$TAG.log
