# edge-tile boxes: parity on mixed interior / edge lattices and the bounds-checked build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "edge_and_interior or rough_ragged or 64cubed or bench_launch" > gpurun_out/t_edges.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_edges.log
timeout 900 python -m pytest tests/test_gpu_memsafety.py -q -m gpu > gpurun_out/t_memsafety.log 2>&1; echo memsafety=$?; tail -2 gpurun_out/t_memsafety.log
