# kernel 3 MLUPS against the state footprint at a fixed 512 x 512 plane (TLB / DRAM-page effects), z-chunk 32
mkdir -p gpurun_out
for rep in 1 2; do
for lat in 512,512,32 512,512,64 512,512,128 512,512,192; do
  timeout 300 python bench.py --lattice $lat --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/fp.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/fp.json'));print('$lat', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], round(d['config']['state_bytes_per_gpu']/1e9,1),'GB')"
done
done
