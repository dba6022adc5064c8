# quick iteration: GPU tests + bench on c5/c3 for the default build, then a variant sweep
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
for cfg in c5 c3; do
  python bench.py --config $cfg --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo bench_$cfg=$?
  python -c "import json;d=json.load(open('gpurun_out/bench_$cfg.json'));r=d['roofline'];print('$cfg', round(d['value']), 'MLUPS', 'k_step', round(r['achieved']), 'GB/s frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3), r['kernel_time_share'])"
done
for v in ${VARIANTS}; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > /dev/null 2>&1 || echo build_fail "$v"
  python bench.py --config c5 --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_v.json'));r=d['roofline'];print('variant $v', round(d['value']), 'MLUPS frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3))"
done
