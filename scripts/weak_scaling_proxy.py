"""Scaling proxy on one GPU.  Weak (default): the per-rank work of the
512^3-at-8-GPUs weak scaling (BASELINE config 5, reading R20: 512 x 512 x 64 per
rank) as P loopback z-slabs of one 512 x 512 x (64 P) lattice with the peer
transport (K_phi edges, device-side epochs, P2P-style pushes into the neighbour
slab, step kernel).  The slabs run one after another on one stream, so time per
step / P is what one rank spends per step on its own GPU, without NVLink latency
or waiting on a neighbour; efficiency proxy E(P) = t(1) / (t(P) / P).
--strong NX NY NZ: the fixed lattice (BASELINE config 4: 256^3) split into P
slabs; a rank's step is t(P) / P, speed-up t(1) / (t(P) / P), E(P) = t(1) / t(P).
  python scripts/weak_scaling_proxy.py STEPS P... [--strong NX NY NZ]
One JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1609_01479_b200 import lb, synth  # noqa: E402

argv = sys.argv[1:]
strong = None
if "--strong" in argv:
    i = argv.index("--strong")
    strong = [int(v) for v in argv[i + 1:i + 4]]
    argv = argv[:i] + argv[i + 4:]
nx, ny, nzr = strong or (512, 512, 64)
steps = int(argv[0]) if argv else 20
ps = [int(v) for v in argv[1:]] or [1, 2, 4, 8]
out = {}
for P in ps:
    nz = nzr if strong else nzr * P
    with lb.Lattice(nx, ny, nz, nslabs=P) as L:
        if P > 1:
            lb.lb_debug_halo_mode(L.h, 1)
        L.init_equilibrium(synth.spinodal_phi(nx, ny, nz, seed=0))
        lb.lb_prepare(L.h)
        st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
        L.step(3)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            L.step(steps)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            best = ms if best is None else min(best, ms)
        lb.lb_profile_reset(L.h)
        lb.lb_profile_enable(L.h, True)
        L.step(steps)
        lb.lb_profile_enable(L.h, False)
        prof = {k: round(v[0] / steps / P, 4) for k, v in lb.lb_profile(L.h).items() if v[1]}
    out[P] = {"ms_per_step": round(best, 4), "ms_per_rank_step": round(best / P, 4),
              "mlups_per_rank": round(nx * ny * (nz // P) / (best / P * 1e-3) / 1e6, 1),
              "kernel_ms_per_rank_step": prof}
if ps[0] == 1:
    for P in ps:
        t1, tp = out[1]["ms_per_step"], out[P]["ms_per_step"]
        out[P]["efficiency_proxy"] = round(t1 / tp if strong else t1 / (tp / P), 4)
        if strong:
            out[P]["speedup_proxy"] = round(t1 / (tp / P), 3)
print(json.dumps({"mode": "strong" if strong else "weak", "lattice" if strong else "per_rank_lattice": [nx, ny, nzr],
                  "transport": "peer (loopback)", "steps": steps, "by_P": out}))
