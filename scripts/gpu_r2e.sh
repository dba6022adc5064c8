# round 2: full GPU suite, CH reorder measurement, variant bench lines
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -rs > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -6 gpurun_out/gpu_tests.log
grep -h "u_strict" gpurun_out/gpu_tests.log | head -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "u_strict or 16cubed" -s > gpurun_out/u_strict.log 2>&1; grep "parity (R18" gpurun_out/u_strict.log | head -8
for c in ch lc mrt; do timeout 600 python bench.py --collision $c --steps 100 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?; head -c 400 gpurun_out/bench_$c.json; echo; done
timeout 600 python bench.py --collision ch --config c3 --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ch_c3.json 2>&1; echo bench_ch_c3=$?; head -c 300 gpurun_out/bench_ch_c3.json; echo
