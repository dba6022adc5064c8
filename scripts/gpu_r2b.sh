# round 2: NEXT-1 device-side epochs + ranks test, L2 policy A/B, bench lines
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
timeout 900 python scripts/ab_tune.py 512 512 64 gt=1 gt=0 gt=3 gt=2 box=0 box=3 box=0,gt=0 ft=0 --rounds 3 > gpurun_out/ab_l2_c5.json 2> gpurun_out/ab_l2_c5.err; echo ab=$?; cat gpurun_out/ab_l2_c5.json; tail -3 gpurun_out/ab_l2_c5.err
timeout 600 python bench.py --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?; cat gpurun_out/bench_default.json
timeout 600 python bench.py --config c3 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3=$?; cat gpurun_out/bench_c3.json | head -c 600; echo
timeout 600 python bench.py --config c5alt --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5alt.json 2> gpurun_out/bench_c5alt.err; echo bench_c5alt=$?; cat gpurun_out/bench_c5alt.json | head -c 600; echo
