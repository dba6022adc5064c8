mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  LB_NVCC_FLAGS="$v" python paper_1609_01479_b200/_build.py --force > gpurun_out/build.log 2>&1 || { echo "build_fail [$v]"; continue; }
  timeout 60 python -c "
from paper_1609_01479_b200 import lb, synth
L = lb.Lattice(64, 64, 16); L.init_equilibrium(synth.spinodal_phi(64, 64, 16))
try:
    lb.lb_debug_step_probe(L.h, 1, 1); print('[$v] probe1 ok')
except Exception as e: print('[$v] probe1 FAIL', str(e)[:100])
" 2>&1 | tail -1
done
