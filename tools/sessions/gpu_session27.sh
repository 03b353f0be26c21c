N="ncu --set full --clock-control none --import-source on"
python tools/prof_gram.py 3 fp32 2000 > /dev/null && $N -k regex:gram_fused_tc -s 1 -c 1 -o gpurun_out/fusedtc2_cfg3 -f python tools/prof_gram.py 3 fp32 2000 > gpurun_out/ncu27a.log 2>&1; echo "a rc=$?"
python tools/prof_gram.py 4 fp64 200 > /dev/null && $N -k regex:gram_mt2 -s 1 -c 1 -o gpurun_out/mt2_cfg4 -f python tools/prof_gram.py 4 fp64 200 > gpurun_out/ncu27b.log 2>&1; echo "b rc=$?"
python tools/prof_gram.py 3 fp64 2000 > /dev/null && $N -k regex:gram_mma -s 1 -c 1 -o gpurun_out/mma_cfg3 -f python tools/prof_gram.py 3 fp64 2000 > gpurun_out/ncu27c.log 2>&1; echo "c rc=$?"
