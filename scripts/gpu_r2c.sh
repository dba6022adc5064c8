# round 2: memory-safety tests (guards + bounds-checked build), rank test, ncu of the ws kernel at c5
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_memsafety.py tests/test_gpu_ranks.py -q -m gpu > gpurun_out/gpu_memsafe.log 2>&1; echo memsafe=$?; tail -3 gpurun_out/gpu_memsafe.log
LB_VARIANT=checked timeout 600 python scripts/sanitize_cases.py > gpurun_out/sanitize_checked.log 2>&1; echo sancheck=$?; tail -4 gpurun_out/sanitize_checked.log
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu_launches=$?
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_kstep_c5 $CMD > gpurun_out/ncu2.log 2>&1; echo ncu_full=$?
