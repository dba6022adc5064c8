"""One step-kernel launch per setting (lb_debug_tune), for ncu's per-launch DRAM
bytes: run under
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_step ...
The launches come in the order of the settings given (after 2 untimed steps of
the defaults).  python scripts/ncu_variants.py NX NY NZ "gt=1" "gt=0" ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1609_01479_b200 import lb, synth  # noqa: E402

KEYS = {"zc": lb.LB_TUNE_ZCHUNK, "band": lb.LB_TUNE_BAND_ROWS, "resid": lb.LB_TUNE_RESID,
        "box": lb.LB_TUNE_L2_BOX, "ft": lb.LB_TUNE_L2_FTILE, "gt": lb.LB_TUNE_L2_GTILE}
DEFAULTS = {"zc": 0, "band": 1, "resid": 0, "box": 2, "ft": 1, "gt": 1}
nx, ny, nz = (int(v) for v in sys.argv[1:4])
with lb.Lattice(nx, ny, nz) as L:
    lb.lb_debug_tune(L.h, lb.LB_TUNE_GRAPHS, 0)
    L.init_equilibrium(synth.spinodal_phi(nx, ny, nz, seed=0))
    L.step(2)
    for s in sys.argv[4:]:
        for kv in s.split(","):
            k, v = kv.split("=")
            lb.lb_debug_tune(L.h, KEYS[k], int(v))
        L.step(1)
        print("launched", s, flush=True)
        for kv in s.split(","):
            k, _ = kv.split("=")
            lb.lb_debug_tune(L.h, KEYS[k], DEFAULTS[k])
