# round-end evidence, part A: GPU suite, smoke, bench lines for every config and variant
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 600 python bench.py --config c3 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
timeout 600 python bench.py --config c2 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null
timeout 600 python bench.py --config c5alt --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5alt.json 2>/dev/null
for c in mrt ch lc; do timeout 600 python bench.py --collision $c --steps 100 --warmup 5 > gpurun_out/bench_$c.json 2>/dev/null; done
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null
for f in default c3 c2 c4 c5alt mrt ch lc; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); r=d['roofline']; print('$f', round(d['value'],1), round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
