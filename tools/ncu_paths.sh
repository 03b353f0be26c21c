#!/bin/bash
# ncu --set full captures of the non-bench kernels (one launch each), after plain runs.
mkdir -p gpurun_out
run() { # tag cfg prec drops regex
  python tools/prof_gram.py $2 $3 $4 > gpurun_out/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$5 -s 1 -c 1 -o gpurun_out/$1 -f \
      python tools/prof_gram.py $2 $3 $4 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
run stream5 5 mat32 16 gram_stream_tc
run ftc3 3 fp32 1000 gram_fused_tc
run mt5 5 fp64 8 gram_mma_tiled
run mma3 3 fp64 1000 gram_mma_kernel
