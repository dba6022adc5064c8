# round-2 full check: GPU suite, smoke, bench lines (default, c3, c4, c5alt, mrt, ch, lc, reference), ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 600 python bench.py --config c3 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; echo bench_c3=$?
timeout 600 python bench.py --config c2 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null; echo bench_c2=$?
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; echo bench_c4=$?
timeout 600 python bench.py --config c5alt --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5alt.json 2>/dev/null; echo bench_c5alt=$?
for c in mrt ch lc; do timeout 600 python bench.py --collision $c --steps 100 --warmup 5 > gpurun_out/bench_$c.json 2>/dev/null; echo bench_$c=$?; done
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null; echo ref=$?
for f in default c3 c2 c4 c5alt mrt ch lc ref; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); r=d.get('roofline') or {}; print('$f', round(d['value'],1), round(r.get('frac',0),4), (d.get('clocks') or {}).get('sm_mhz'))"; done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu_launches=$?
