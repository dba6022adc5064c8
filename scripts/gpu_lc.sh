# NEXT-4 liquid-crystal path: GPU parity, bench line, launch list and one ncu --set full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lc.py -q > gpurun_out/gpu_tests_lc.log 2>&1; echo tests_lc=$?; tail -3 gpurun_out/gpu_tests_lc.log
timeout 300 python bench.py --collision lc --steps 100 > gpurun_out/bench_lc.json 2> gpurun_out/bench_lc.err; echo bench_lc=$?
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --collision lc --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_lc.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_lc.csv $CMD > gpurun_out/ncu1_lc.log 2>&1; echo ncu_launches=$?
$CMD > gpurun_out/plain2_lc.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_lc -s 3 -c 1 -o gpurun_out/prof_kstep_lc $CMD > gpurun_out/ncu2_lc.log 2>&1; echo ncu_full=$?
