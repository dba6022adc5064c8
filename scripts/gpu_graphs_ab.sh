# step time with and without CUDA graphs (the per-launch profile region runs without)
mkdir -p gpurun_out
timeout 600 python scripts/ab_tune.py 512 512 64 "graphs=1" "graphs=0" --rounds 4 --steps 40 > gpurun_out/ab_graphs.txt 2>&1
timeout 600 python scripts/ab_tune.py 128 128 128 "graphs=1" "graphs=0" --rounds 4 --steps 200 >> gpurun_out/ab_graphs.txt 2>&1
cat gpurun_out/ab_graphs.txt
