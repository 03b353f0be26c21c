mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_s11.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_s11.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s11.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_s11.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_s11.json 2>gpurun_out/bench_s11.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_s11.json'));print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
