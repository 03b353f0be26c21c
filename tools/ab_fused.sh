# A/B of fused fp32 variants on the GPU box: bash tools/ab_fused.sh NAME...
for v in "$@"; do
  python tools/variants.py time $v 5 fp32 296 5
  python tools/variants.py time $v 3 fp32 10000 5
  python tools/variants.py time $v 4 fp32 1000 5
done
