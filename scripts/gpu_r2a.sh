# round 2, first check of the cleaned library: GPU tests, smoke, block-order A/B, bench
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 python scripts/ab_tune.py 512 512 64 band=1 band=2 band=4 band=8 band=4,zc=64 band=8,zc=64 band=16,zc=64 --rounds 3 > gpurun_out/ab_band_c5.json 2> gpurun_out/ab_band_c5.err; echo ab=$?; cat gpurun_out/ab_band_c5.json
timeout 600 python scripts/ab_tune.py 256 256 256 band=1 band=4 band=8 band=8,zc=64 --rounds 3 > gpurun_out/ab_band_c4.json 2>&1; echo ab4=$?; cat gpurun_out/ab_band_c4.json
timeout 600 python bench.py --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?; cat gpurun_out/bench_default.json
