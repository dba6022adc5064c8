# phi-exchange lag variants on the one-wave lattices: A/B kernel 3 vs 5 and the c2 bench line
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:- }"
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > /dev/null 2>&1 || echo build_fail "$v"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "xch" > gpurun_out/lag_tests.log 2>&1; echo "[$v] tests=$?"
  for lat in 64,64,64 128,128,128; do
    echo "[$v] lat=$lat $(timeout 300 python scripts/probe.py --lattice $lat --ab 3,5 --steps 50 --rounds 10 2>&1 | tail -1)"
  done
done
