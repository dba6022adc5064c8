"""Interleaved A/B of step kernels (lb_debug_step_kernel) on one lattice and one
handle: MLUPS of each kernel, round-robin over several rounds (the power-capped
clock drifts between runs, so kernels are compared inside one process).

  python scripts/ab_kernels.py NX NY NZ --collision lc --kernels 1 2 [--rounds 4] [--steps 40]
Prints one JSON line: {kernel: [MLUPS per round]}.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1609_01479_b200 import lb, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("nx", type=int)
ap.add_argument("ny", type=int)
ap.add_argument("nz", type=int)
ap.add_argument("--kernels", type=int, nargs="+", default=[1, 2])
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--collision", default="lc", choices=["bgk", "mrt", "ch", "lc"])
a = ap.parse_args()

out = {str(k): [] for k in a.kernels}
if a.collision == "lc":
    L = lb.LcLattice(a.nx, a.ny, a.nz)
    L.init(synth.random_directors(a.nx, a.ny, a.nz, 0))
else:
    L = (lb.ChLattice if a.collision == "ch" else lb.Lattice)(a.nx, a.ny, a.nz)
    if a.collision == "mrt":
        lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
    L.init_equilibrium(synth.spinodal_phi(a.nx, a.ny, a.nz, seed=0))
with L:
    st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    for _ in range(a.rounds):
        for k in a.kernels:
            lb.lb_debug_step_kernel(L.h, k)
            lb.lb_prepare(L.h)
            L.step(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            L.step(a.steps)
            e1.record(st)
            torch.cuda.synchronize()
            out[str(k)].append(round(a.nx * a.ny * a.nz * a.steps / (e0.elapsed_time(e1) * 1e-3) / 1e6, 1))
print(json.dumps({"lattice": [a.nx, a.ny, a.nz], "collision": a.collision, "mlups": out}))
