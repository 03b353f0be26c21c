mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
python tools/prof_sweep.py 2000 > /dev/null && $N -k regex:gram_split -s 1 -c 1 -o gpurun_out/split_cfg2 -f python tools/prof_sweep.py 2000 > gpurun_out/ncu12a.log 2>&1; echo "a rc=$?"
python tools/prof_blk.py 1000 35000 148 >/dev/null && $N -k regex:gram_blk -s 1 -c 1 -o gpurun_out/blk2_k1000 -f python tools/prof_blk.py 1000 35000 148 > gpurun_out/ncu12b.log 2>&1; echo "b rc=$?"
$N -k regex:gram_blk -s 1 -c 1 -o gpurun_out/blk2_k100 -f python tools/prof_blk.py 100 35000 1000 > gpurun_out/ncu12c.log 2>&1; echo "c rc=$?"
python tools/prof_app_a.py 1000 148 > /dev/null && $N -k regex:chol -s 1 -c 1 -o gpurun_out/chol_k1000 -f python tools/prof_app_a.py 1000 148 > gpurun_out/ncu12d.log 2>&1; echo "d rc=$?"
$N -k regex:chol -s 1 -c 1 -o gpurun_out/chol_k100 -f python tools/prof_app_a.py 100 2000 > gpurun_out/ncu12e.log 2>&1; echo "e rc=$?"
python tools/prof_gram.py 3 fp32 2000 > /dev/null && $N -k regex:gram_fused_tc -s 1 -c 1 -o gpurun_out/fusedtc_cfg3 -f python tools/prof_gram.py 3 fp32 2000 > gpurun_out/ncu12f.log 2>&1; echo "f rc=$?"
