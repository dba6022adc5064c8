mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
run() {
  local lab=$1; shift
  env $ENVV timeout 300 python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));print('$lab', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$lab failed"
}
run c5 --steps 100
run c3 --config c3 --steps 100
run c2 --config c2 --steps 1000
run c4 --config c4 --steps 50
run ch_c5 --collision ch --steps 100
run ch_c3 --collision ch --config c3 --steps 100
ENVV="LB_TILE_ROWS=4" run ch_c3_ty4 --collision ch --config c3 --steps 100
run lc_c3_default --collision lc --config c3 --steps 100
ENVV="LB_ZCHUNK=64" run lc_c3_zc64 --collision lc --config c3 --steps 100
ENVV="LB_ZCHUNK=32" run lc_c3_zc32 --collision lc --config c3 --steps 100
ENVV="LB_ZCHUNK=32" run lc_c5_zc32 --collision lc --steps 100
run lc_c5 --collision lc --steps 100
