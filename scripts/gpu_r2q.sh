mkdir -p gpurun_out
python -c "from paper_1609_01479_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
python scripts/kphi_probe.py > gpurun_out/kphi_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_phi_edges -s 2 -c 1 -o gpurun_out/prof_kphi python scripts/kphi_probe.py > gpurun_out/ncu_kphi.log 2>&1; echo ncu=$?
