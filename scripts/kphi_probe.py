"""A few steps of 512 x 512 x 64 as two loopback slabs with the peer transport
(for ncu on k_phi_edges)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1609_01479_b200 import lb, synth  # noqa: E402

with lb.Lattice(512, 512, 64, nslabs=2) as L:
    lb.lb_debug_tune(L.h, lb.LB_TUNE_GRAPHS, 0)
    L.init_equilibrium(synth.spinodal_phi(512, 512, 64, seed=0))
    L.step(4)
print("ok")
