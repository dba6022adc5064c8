# bench lines after the roofline-basis change (value region per launch where a step is one kernel)
mkdir -p gpurun_out
timeout 600 python bench.py --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 600 python bench.py --config c3 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
timeout 600 python bench.py --config c2 --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null
timeout 600 python bench.py --config c5alt --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5alt.json 2>/dev/null
for c in mrt ch lc; do timeout 600 python bench.py --collision $c --steps 100 --warmup 5 > gpurun_out/bench_$c.json 2>/dev/null; done
for f in default c3 c2 c4 c5alt mrt ch lc; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json')); r=d['roofline']; print('$f', round(d['value'],1), round(r['frac'],4), round(r['avg_launch_ms'],4), round(r['avg_launch_ms_evented'],4), r['avg_launch_basis'][:20], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
