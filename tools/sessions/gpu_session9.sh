mkdir -p gpurun_out
python tools/prof_blk.py 1000 35000 148 && \
ncu --set full --clock-control none --import-source on -k regex:gram_blk -s 1 -c 1 -o gpurun_out/blk_k1000 -f python tools/prof_blk.py 1000 35000 148 > gpurun_out/ncu_blk_k1000.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gram_blk -s 1 -c 1 -o gpurun_out/blk_k100 -f python tools/prof_blk.py 100 35000 1000 > gpurun_out/ncu_blk_k100.log 2>&1; echo "ncu2 rc=$?"
