mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True); _build.build(force=True, checked=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ch.py -q -m gpu -x > gpurun_out/t_ch.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_ch.log
timeout 300 python scripts/ab_tune.py 512 512 64 zc=0 --kernel 2 --collision ch --rounds 3 > gpurun_out/ab_chws.json 2>&1; cat gpurun_out/ab_chws.json
timeout 300 python scripts/ab_tune.py 128 128 128 zc=0 --kernel 2 --collision ch --rounds 2 > gpurun_out/ab_chws3.json 2>&1; cat gpurun_out/ab_chws3.json
