# build-variant sweep (variants separated by ';') of the interleaved A/B timing of
# step kernels 1 (tile) and 3 (warp-specialised); GPU tests on the default build first
mkdir -p gpurun_out
python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo build_fail; tail gpurun_out/build.log; }
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log; fi
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > /dev/null 2>&1 || echo build_fail
  for cfg in ${CFGS:-c5 c3}; do
    timeout 300 python scripts/probe.py --config $cfg --ab ${AB:-1,3} --steps 10 --rounds ${ROUNDS:-20} > gpurun_out/ab.json 2>&1
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('[$v]', '$cfg', {k:round(x['mlups']) for k,x in d.items() if k.startswith('ab')})" || tail -3 gpurun_out/ab.json
  done
done
