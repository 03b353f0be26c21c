for nt in 192 5 192 5; do
  XLMIMO_GRAM_NT=$nt timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b30_$nt.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b30_$nt.json'));r=d['roofline'];print('$nt', round(d['ms_per_step'],3), round(r['launch_ms'],3), round(r['frac'],4))"
done
