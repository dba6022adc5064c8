# c3 (128^3) tile-shape / z-chunk / kernel sweep with bench.py, interleaved rounds
mkdir -p gpurun_out
run() {  # label env...
  local lab=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c3} --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$lab', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" || echo "$lab failed"
}
for i in 1 2; do
  run default X=1
  run ty8_zc64 LB_TILE_ROWS=8 LB_ZCHUNK=64
  run ty8_zc43 LB_TILE_ROWS=8 LB_ZCHUNK=43
  run ty8_zc32 LB_TILE_ROWS=8 LB_ZCHUNK=32
  run ty4_zc32 LB_TILE_ROWS=4 LB_ZCHUNK=32
  run ty4_zc64 LB_TILE_ROWS=4 LB_ZCHUNK=64
done
