# c5 bench under tile_of_block group sizes (LB_RESID), alternated A B A B
mkdir -p gpurun_out
for rep in 1 2; do
  for r in 148 144 128 296 74 1024; do
    LB_RESID=$r timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/resid.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/resid.json'));print('resid $r', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
