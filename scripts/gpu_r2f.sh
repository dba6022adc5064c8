# CH tile rows A/B; ranks NCCL test; tune tests
mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ch.py tests/test_gpu_ranks.py tests/test_gpu_parity.py -q -m gpu -k "tile_rows or ranks or nccl or tune or u_strict or 16cubed" -s > gpurun_out/t_f.log 2>&1; echo tests=$?; grep -E "passed|failed|lb_create_slab, two" gpurun_out/t_f.log | tail -3
timeout 600 python scripts/ab_tune.py 512 512 64 ty=8 ty=4 --collision ch --rounds 3 > gpurun_out/ab_ch_ty.json 2>&1; echo ab=$?; cat gpurun_out/ab_ch_ty.json
timeout 600 python scripts/ab_tune.py 128 128 128 ty=8 ty=4 --collision ch --rounds 3 > gpurun_out/ab_ch_ty_c3.json 2>&1; echo ab3=$?; cat gpurun_out/ab_ch_ty_c3.json
