mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_gr -s 3 -c 1 -o gpurun_out/prof_kstep_gr $CMD > gpurun_out/ncu_gr.log 2>&1; echo ncu=$?
