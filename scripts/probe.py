"""Memory-side ceiling of the step kernel: time lb_step against the two
lb_debug_step_probe modes (same copies and stores, no physics) and a plain
device copy, at one BASELINE config.  Prints one JSON line.

  python scripts/probe.py [--config c5] [--steps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1609_01479_b200 import lb, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    nx, ny, nzf, _, desc = bench.CONFIGS[a.config]
    nz = nzf(1)
    L = lb.Lattice(nx, ny, nz)
    L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
    stream = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    out = {"config": a.config, "sites": nx * ny * nz}

    def timed(fn):
        fn(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(a.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        return {"ms_per_step": ms, "mlups": nx * ny * nz / ms / 1e3, "gbs_608": nx * ny * nz * 608 / ms / 1e6}

    out["step"] = timed(lambda n: L.step(n))
    out["probe1_copy_push"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 1))
    out["probe2_plus_halo_phi_P"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 2))
    out["probe3_tile_only"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 3))
    out["k_stream_site_parallel"] = timed(lambda n: lb.lb_debug_stream(L.h, n))
    n = nx * ny * nz * 38
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    y.copy_(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out["torch_copy_same_bytes"] = {"ms": ms, "gbs": 2 * n * 8 / ms / 1e6}
    L.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
