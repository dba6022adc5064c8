mkdir -p gpurun_out
LB_VARIANT=fldg timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "16cubed or ws_kernel or 64cubed_10" > gpurun_out/t_fldg.log 2>&1; echo tests_fldg=$?; tail -2 gpurun_out/t_fldg.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "edge_chunks or slabs_parity or tune" > gpurun_out/t_edge.log 2>&1; echo tests_edge=$?; tail -2 gpurun_out/t_edge.log
bash scripts/ab_builds.sh fldg "" 4 --steps 100 --warmup 5 > gpurun_out/ab_fldg.txt 2>&1; cat gpurun_out/ab_fldg.txt
