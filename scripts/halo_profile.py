"""Loopback z-slabs of 512 x 512 x 64 with the peer transport (K_phi edges + the
step kernel, ordered by the device-side epochs): per-kernel device time from
lb_profile (CUDA events around each launch) and MLUPS with graphs; one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1609_01479_b200 import lb, synth  # noqa: E402

nx, ny, nz = 512, 512, 64
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
phi = synth.spinodal_phi(nx, ny, nz, seed=0)
out = {}
for nslabs, halo in ((1, None), (2, 1), (4, 1), (8, 1), (2, 0), (4, 0)):
    with lb.Lattice(nx, ny, nz, nslabs=nslabs) as L:
        if halo is not None:
            lb.lb_debug_halo_mode(L.h, halo)
        L.init_equilibrium(phi)
        lb.lb_prepare(L.h)
        st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
        L.step(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = lb.lb_launch_count(L.h)
        e0.record(st)
        L.step(steps)
        e1.record(st)
        torch.cuda.synchronize()
        mlups = nx * ny * nz * steps / (e0.elapsed_time(e1) * 1e-3) / 1e6
        launches = lb.lb_launch_count(L.h) - n0
        lb.lb_profile_reset(L.h)
        lb.lb_profile_enable(L.h, True)
        L.step(steps)
        lb.lb_profile_enable(L.h, False)
        prof = {k: {"ms_per_step": round(v[0] / steps, 4), "launches_per_step": v[1] / steps}
                for k, v in lb.lb_profile(L.h).items() if v[1]}
        assert lb.lb_debug_guards(L.h) == 0
        key = f"{nslabs} slab(s)" + ("" if halo is None else (" peer" if halo == 1 else " exchange"))
        out[key] = {"mlups": round(mlups, 1), "kernel_launches_per_step": launches / steps, "profile": prof}
print(json.dumps(out))
