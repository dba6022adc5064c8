mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
CMD="python bench.py --collision ch --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_ch.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_ch -s 3 -c 1 -o gpurun_out/prof_kstep_chws2 $CMD > gpurun_out/ncu_ch.log 2>&1; echo ncu=$?
