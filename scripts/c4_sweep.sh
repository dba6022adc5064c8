mkdir -p gpurun_out
run() {
  local cfg=$1 lab=$2; shift 2
  env "$@" timeout 300 python bench.py --config $cfg --steps ${STEPS:-50} --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$cfg $lab', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$cfg $lab failed"
}
for i in 1 2; do
  run c4 default X=1
  run c4 ty8_zc256 LB_TILE_ROWS=8 LB_ZCHUNK=256
  run c4 ty8_zc128 LB_TILE_ROWS=8 LB_ZCHUNK=128
  run c4 ty8_zc64 LB_TILE_ROWS=8 LB_ZCHUNK=64
  run c4 ty8_zc32 LB_TILE_ROWS=8 LB_ZCHUNK=32
  run c4 ty4_zc64 LB_TILE_ROWS=4 LB_ZCHUNK=64
done
