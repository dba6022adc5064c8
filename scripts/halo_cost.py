"""Cost of the slab decomposition on one GPU (loopback): MLUPS of the whole
512x512x64 lattice as 1 slab, and as 2 / 4 slabs with the fused (peer) halo and
with the exchange transport.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1609_01479_b200 import lb, synth  # noqa: E402

nx, ny, nz = 512, 512, 64
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
phi = synth.spinodal_phi(nx, ny, nz)
out = {}
for nslabs, halo in ((1, None), (2, 1), (2, 0), (4, 1), (4, 0), (8, 1), (8, 0)):
    with lb.Lattice(nx, ny, nz, nslabs=nslabs) as L:
        if halo is not None:
            lb.lb_debug_halo_mode(L.h, halo)
        L.init_equilibrium(phi)
        st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
        L.step(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.step(steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[f"slabs{nslabs}_{'peer' if halo == 1 else ('exchange' if halo == 0 else 'none')}"] = round(
            nx * ny * nz / ms / 1e3)
print(json.dumps(out))
