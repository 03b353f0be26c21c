#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for c in 0 1 2 3; do
  XLMIMO_SPLIT_CFG=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2>gpurun_out/bench_cfg$c.err
  echo "cfg $c: $(python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));print(d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['frac'], d['clocks'])")"
done
bash tools/ncu_gram.sh split 2000 gram_split
