# warp-specialised kernel: its GPU tests, then probe timings at c5 / c3 (bounded by timeout)
mkdir -p gpurun_out
python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo build_fail; tail gpurun_out/build.log; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ws" > gpurun_out/ws_tests.log 2>&1; echo ws_tests=$?; tail -5 gpurun_out/ws_tests.log
for cfg in c5 c3 c2; do
  timeout 300 python scripts/probe.py --config $cfg --steps 50 > gpurun_out/probe_$cfg.json 2>gpurun_out/probe_$cfg.err; echo probe_$cfg=$?
  python -c "import json;d=json.load(open('gpurun_out/probe_$cfg.json'));print('$cfg', {k:(round(v['mlups']) if isinstance(v,dict) and 'mlups' in v else v) for k,v in d.items()})" 2>/dev/null || tail -3 gpurun_out/probe_$cfg.err
done
