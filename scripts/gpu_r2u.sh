mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True); _build.build(force=True, checked=True)" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "ws_kernel or 16cubed" > gpurun_out/t_gr1.log 2>&1; echo tests1=$?; tail -4 gpurun_out/t_gr1.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py tests/test_gpu_ranks.py -q -m gpu > gpurun_out/t_gr.log 2>&1; echo tests=$?; tail -4 gpurun_out/t_gr.log
timeout 400 python scripts/ab_tune.py 512 512 64 var=0 var=1 --rounds 4 > gpurun_out/ab_gr_c5.json 2>&1; cat gpurun_out/ab_gr_c5.json
timeout 400 python scripts/ab_tune.py 256 256 256 var=0 var=1 --rounds 3 > gpurun_out/ab_gr_c4.json 2>&1; cat gpurun_out/ab_gr_c4.json
