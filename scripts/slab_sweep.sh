mkdir -p gpurun_out
run() {
  local lat=$1 lab=$2; shift 2
  env "$@" timeout 300 python bench.py --lattice $lat --steps ${STEPS:-50} --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$lat $lab', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$lat $lab failed"
}
for i in 1 2; do
  run 256,256,32 default X=1
  run 256,256,32 ty8_zc32 LB_TILE_ROWS=8 LB_ZCHUNK=32
  run 256,256,32 ty8_zc16 LB_TILE_ROWS=8 LB_ZCHUNK=16
  run 256,256,32 ty8_zc8 LB_TILE_ROWS=8 LB_ZCHUNK=8
  run 256,256,64 ty8_zc32 LB_TILE_ROWS=8 LB_ZCHUNK=32
  run 256,256,64 ty8_zc16 LB_TILE_ROWS=8 LB_ZCHUNK=16
  run 256,256,256 ty8_zc16 LB_TILE_ROWS=8 LB_ZCHUNK=16
  STEPS=200 run 128,128,64 ty8_zc32 LB_TILE_ROWS=8 LB_ZCHUNK=32
  STEPS=200 run 128,128,64 ty8_zc16 LB_TILE_ROWS=8 LB_ZCHUNK=16
  STEPS=200 run 128,128,64 default X=1
done
