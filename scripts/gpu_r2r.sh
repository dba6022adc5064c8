mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True); _build.build(force=True, checked=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranks.py -q -m gpu -x -k "slab or fused or graph or rank or nccl" > gpurun_out/t_p.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_p.log
timeout 600 python scripts/halo_profile.py 40 > gpurun_out/halo_profile.json 2>&1; echo halo=$?; python -c "
import json; d=json.load(open('gpurun_out/halo_profile.json'))
for k,v in d.items(): print(k, v['mlups'], v['profile'].get('k_phi'))"
python scripts/kphi_probe.py > gpurun_out/kphi_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_phi_edges -s 2 -c 1 -o gpurun_out/prof_kphi2 python scripts/kphi_probe.py > gpurun_out/ncu_kphi.log 2>&1; echo ncu=$?
