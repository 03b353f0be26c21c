mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b16.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s16.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_s16.log 2>&1; echo "launch rc=$?"
python tools/prof_sweep.py 10000 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:gram_split -s 1 -c 1 \
    -o gpurun_out/split_bench_d10000 -f python tools/prof_sweep.py 10000 > gpurun_out/ncu16b.log 2>&1; echo "full rc=$?"
