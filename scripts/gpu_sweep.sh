# build-variant sweep: bench c5 and c3 for each LB_NVCC_FLAGS variant (separated by ';')
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo "build_fail [$v]"; tail -5 gpurun_out/build.log; continue; }
  for cfg in ${CFGS:-c5 c3}; do
    python bench.py --config $cfg --steps ${STEPS:-100} --no-cpu-baseline --no-e2e > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err || { echo "bench_fail [$v] $cfg"; tail -3 gpurun_out/bench_v.err; continue; }
    python -c "import json;d=json.load(open('gpurun_out/bench_v.json'));r=d['roofline'];print('[$v] $cfg', round(d['value']), 'MLUPS frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))"
  done
done
