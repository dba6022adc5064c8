mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True); _build.build(force=True, checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranks.py tests/test_gpu_memsafety.py -q -m gpu -x > gpurun_out/t_o.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_o.log
timeout 600 python scripts/halo_profile.py 40 > gpurun_out/halo_profile.json 2>&1; echo halo=$?; cat gpurun_out/halo_profile.json
bash scripts/ab_builds.sh old "" 3 --steps 100 --warmup 5 > gpurun_out/ab_makephi.txt 2>&1; cat gpurun_out/ab_makephi.txt
