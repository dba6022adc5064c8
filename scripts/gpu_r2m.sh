# BOX2 ws kernel: parity suite, A/B against the one-box kernel (variant 1)
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True); _build.build(force=True, checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memsafety.py -q -m gpu -x > gpurun_out/t_par.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_par.log
timeout 400 python scripts/ab_tune.py 512 512 64 var=0 var=1 --rounds 4 > gpurun_out/ab_box2_c5.json 2>&1; cat gpurun_out/ab_box2_c5.json
timeout 400 python scripts/ab_tune.py 256 256 256 var=0 var=1 --rounds 3 > gpurun_out/ab_box2_c4.json 2>&1; cat gpurun_out/ab_box2_c4.json
