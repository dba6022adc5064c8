# round-end evidence: GPU suite, smoke, bench lines for every config and variant, ncu
# launch lists and one --set full capture per step kernel (scripts/update_profiles.py r2)
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
run_ncu() {  # name, kernel regex, bench args
  CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $3"
  $CMD > gpurun_out/plain_$1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$1.csv $CMD > gpurun_out/ncu1_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o gpurun_out/prof_kstep_$1 $CMD > gpurun_out/ncu2_$1.log 2>&1; echo ncu_$1=$?
}
run_ncu c5 k_step_ws ""
run_ncu c3 k_step_ws "--config c3"
run_ncu c2 k_step_ws "--config c2"
run_ncu c4 k_step_ws "--config c4"
run_ncu mrt k_step_ws "--collision mrt"
run_ncu ch k_step_ch "--collision ch"
run_ncu lc k_step_lc "--collision lc"
mv gpurun_out/launches_c5.csv gpurun_out/launches.csv
