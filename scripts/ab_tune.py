"""Interleaved A/B of step-kernel launch knobs (lb_debug_tune) on one lattice:
MLUPS of each setting, measured round-robin over several rounds (the power-capped
clock drifts between runs, so settings are compared inside one process).

  python scripts/ab_tune.py NX NY NZ "band=1" "band=4" "band=4,zc=64" ... [--rounds 3] [--steps 40] [--kernel K]
Prints one JSON line: {setting: [MLUPS per round]}.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1609_01479_b200 import lb, synth  # noqa: E402

KEYS = {"zc": lb.LB_TUNE_ZCHUNK, "band": lb.LB_TUNE_BAND_ROWS, "resid": lb.LB_TUNE_RESID, "graphs": lb.LB_TUNE_GRAPHS,
        "box": lb.LB_TUNE_L2_BOX, "ft": lb.LB_TUNE_L2_FTILE, "gt": lb.LB_TUNE_L2_GTILE, "ty": lb.LB_TUNE_TILE_ROWS,
        "var": lb.LB_TUNE_VARIANT}
DEFAULTS = {"zc": 0, "band": 1, "resid": 0, "graphs": 1, "box": 2, "ft": 1, "gt": 1, "ty": 0, "var": 0}

ap = argparse.ArgumentParser()
ap.add_argument("nx", type=int)
ap.add_argument("ny", type=int)
ap.add_argument("nz", type=int)
ap.add_argument("settings", nargs="+")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--collision", default="bgk")
a = ap.parse_args()

phi = synth.spinodal_phi(a.nx, a.ny, a.nz, seed=0)
out = {s: [] for s in a.settings}
Lat = lb.ChLattice if a.collision == "ch" else lb.Lattice
with Lat(a.nx, a.ny, a.nz) as L:
    lb.lb_debug_step_kernel(L.h, a.kernel)
    if a.collision == "mrt":
        lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
    L.init_equilibrium(phi)
    st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    for _ in range(a.rounds):
        for s in a.settings:
            for kv in s.split(","):
                k, v = kv.split("=")
                lb.lb_debug_tune(L.h, KEYS[k], int(v))
            lb.lb_prepare(L.h)
            L.step(3)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            L.step(a.steps)
            e1.record(st)
            torch.cuda.synchronize()
            out[s].append(round(a.nx * a.ny * a.nz * a.steps / (e0.elapsed_time(e1) * 1e-3) / 1e6, 1))
            for kv in s.split(","):  # back to the defaults
                k, _ = kv.split("=")
                lb.lb_debug_tune(L.h, KEYS[k], DEFAULTS[k])
print(json.dumps({"lattice": [a.nx, a.ny, a.nz], "kernel": a.kernel, "mlups": out}))
