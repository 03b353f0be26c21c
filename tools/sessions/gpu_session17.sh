mkdir -p gpurun_out
XLMIMO_GRAM_NT=1192 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "sweep or determinism" > gpurun_out/pytest_s17.log 2>&1; echo "pytest(pipe) rc=$?"; tail -1 gpurun_out/pytest_s17.log
for nt in 192 1192 1128 1256 192; do
  XLMIMO_GRAM_NT=$nt timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b17_$nt.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b17_$nt.json'));r=d['roofline'];print('$nt', round(d['ms_per_step'],3), round(r['launch_ms'],3), round(r['frac'],4), d['clocks']['sm_mhz'])"
done
