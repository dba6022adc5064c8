# full round check: GPU tests, smoke, bench lines, reference arm, ncu launch lists + full captures
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 300 python bench.py --config c3 --steps 2000 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; echo bench_c3=$?
timeout 300 python bench.py --config c2 --steps 1000 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null; echo bench_c2=$?
timeout 300 python bench.py --config c4 --steps 50 --no-cpu-baseline > gpurun_out/bench_c4.json 2>/dev/null; echo bench_c4=$?
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>/dev/null; echo ref=$?
timeout 300 python bench.py --collision mrt --steps 100 > gpurun_out/bench_mrt.json 2>/dev/null; echo bench_mrt=$?
timeout 300 python bench.py --collision ch --steps 100 > gpurun_out/bench_ch.json 2>/dev/null; echo bench_ch=$?
timeout 300 python bench.py --collision lc --steps 100 > gpurun_out/bench_lc.json 2>/dev/null; echo bench_lc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu_launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_kstep_c5 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu_full=$?
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu1_c3.log 2>&1; echo ncu_launches_c3=$?
$CMD > gpurun_out/plain2_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_kstep_c3 $CMD > gpurun_out/ncu2_c3.log 2>&1; echo ncu_full_c3=$?
CMD="python bench.py --collision lc --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_lc.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_lc.csv $CMD > gpurun_out/ncu1_lc.log 2>&1; echo ncu_launches_lc=$?
$CMD > gpurun_out/plain2_lc.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_lc -s 3 -c 1 -o gpurun_out/prof_kstep_lc $CMD > gpurun_out/ncu2_lc.log 2>&1; echo ncu_full_lc=$?
