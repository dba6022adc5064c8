# CH block order (chunk after chunk of a tile): parity, A/B against the previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ch.py -q -m gpu -x > gpurun_out/t_ad.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_ad.log
bash scripts/ab_builds.sh old "" 3 --collision ch --steps 200 > gpurun_out/ab_chorder_c5.txt 2>&1
bash scripts/ab_builds.sh old "" 2 --collision ch --config c4 --steps 200 > gpurun_out/ab_chorder_c4.txt 2>&1
cat gpurun_out/ab_chorder_*.txt
