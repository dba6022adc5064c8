"""Where the warp-specialised kernel differs from the tile kernel (debug)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import lb_ref as R  # noqa: E402
from paper_1609_01479_b200 import lb, synth  # noqa: E402

for shape in [(16, 16, 16), (64, 64, 16), (34, 10, 7)]:
    nx, ny, nz = shape
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, 14)
    f, g = R.equilibrium_state(rho, u, phi, R.Params())
    f, g = f + nf, g + ng
    out = []
    for k in (1, 3):
        with lb.Lattice(nx, ny, nz) as L:
            lb.lb_debug_step_kernel(L.h, k)
            L.set_state(f, g)
            L.step(1)
            out.append(L.get_state())
    for name, a, b in (("f", out[0][0], out[1][0]), ("g", out[0][1], out[1][1])):
        d = np.abs(a - b)
        bad = np.argwhere(d > 0)
        print(shape, name, "maxdiff", d.max(), "nbad", len(bad), "of", d.size, "first", bad[:5].tolist(),
              "rel", d.max() / np.abs(a).max())
        if len(bad):
            zs = sorted(set(bad[:, 1].tolist()))
            ys = sorted(set(bad[:, 2].tolist()))
            xs = sorted(set(bad[:, 3].tolist()))
            print("   comps", sorted(set(bad[:, 0].tolist())), "z", zs[:20], "y", ys[:20], "x", xs[:40])
