"""Short run for ncu: one launch each of the step kernel (tile), its probe modes
1-4, and the warp-specialised step kernel, after warm-up."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1609_01479_b200 import lb, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
nx, ny, nzf, _, _ = bench.CONFIGS[cfg]
nz = nzf(1)
L = lb.Lattice(nx, ny, nz)
L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
lb.lb_debug_step_kernel(L.h, 1)
L.step(2)
L.step(1)
for mode in (1, 2, 3, 4):
    lb.lb_debug_step_probe(L.h, 1, mode)
lb.lb_debug_step_kernel(L.h, 3)
L.step(1)
L.close()
L = lb.ChLattice(nx, ny, nz)
L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
L.step(2)
L.close()
print("ok")
