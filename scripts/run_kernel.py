"""Run lb_step with one step kernel (lb_debug_step_kernel) at a bench config, for
ncu captures:  python scripts/run_kernel.py --config c3 --kernel 5 --steps 4"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_01479_b200 import lb, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--lattice", default="", help="NX,NY,NZ instead of the config's lattice")
a = ap.parse_args()
nx, ny, nzf, _, _ = bench.CONFIGS[a.config]
nz = nzf(1)
if a.lattice:
    nx, ny, nz = (int(v) for v in a.lattice.split(","))
L = lb.Lattice(nx, ny, nz)
L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
lb.lb_debug_step_kernel(L.h, a.kernel)
for _ in range(a.steps):
    L.step(1)
torch.cuda.synchronize()
L.close()
print("done")
