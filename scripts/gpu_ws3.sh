mkdir -p gpurun_out
python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo build_fail; tail gpurun_out/build.log; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
VARIANTS="-DLB_STEP_WAVES=8;-DLB_STEP_WAVES=4;-DLB_STEP_WAVES=16" REPEAT=3 PROBE_ONLY=step_ws,step_tile CFGS="c5 c3" bash scripts/gpu_probe_sweep.sh
