# c5 / c2 z-chunk and tile-shape sweep with bench.py (interleaved)
mkdir -p gpurun_out
run() {  # cfg label env...
  local cfg=$1 lab=$2; shift 2
  env "$@" timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$cfg $lab', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$cfg $lab failed"
}
for i in 1 2; do
  run c5 default X=1
  run c5 zc64 LB_ZCHUNK=64
  run c5 zc16 LB_ZCHUNK=16
done
for i in 1 2; do
  STEPS=1000 run c2 default X=1
  STEPS=1000 run c2 ty8_zc8 LB_TILE_ROWS=8 LB_ZCHUNK=8
  STEPS=1000 run c2 ty8_zc16 LB_TILE_ROWS=8 LB_ZCHUNK=16
  STEPS=1000 run c2 ty4_zc16 LB_TILE_ROWS=4 LB_ZCHUNK=16
done
