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
    ap.add_argument("--only", default="", help="comma-separated subset of the timings")
    ap.add_argument("--ab", default="", help="interleaved A/B of step kernels, e.g. 1,3 (lb_debug_step_kernel)")
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--mrt", action="store_true", help="collision model 1 (stress in f^eq, MRT)")
    ap.add_argument("--ch", action="store_true", help="the finite-difference Cahn-Hilliard variant (lb_create_ch)")
    ap.add_argument("--lattice", default="", help="NX,NY,NZ instead of the config's lattice")
    a = ap.parse_args()
    nx, ny, nzf, _, desc = bench.CONFIGS[a.config]
    nz = nzf(1)
    if a.lattice:
        nx, ny, nz = (int(v) for v in a.lattice.split(","))
    if a.ch:
        L = lb.ChLattice(nx, ny, nz)
        L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
        st = torch.cuda.ExternalStream(lb.lb_stream(L.h))
        L.step(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.step(a.steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        print(json.dumps({"config": a.config, "ch_mlups": nx * ny * nz / ms / 1e3, "gbs_320": nx * ny * nz * 320 / ms / 1e6}))
        L.close()
        return
    L = lb.Lattice(nx, ny, nz)
    L.init_equilibrium(synth.spinodal_phi(nx, ny, nz))
    stream = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    if a.mrt:
        lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
    out = {"config": a.config, "sites": nx * ny * nz}

    only = set(a.only.split(",")) if a.only else None

    def timed(fn, name=None):
        if only is not None and name not in only:
            return None
        fn(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(a.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        return {"ms_per_step": ms, "mlups": nx * ny * nz / ms / 1e3, "gbs_608": nx * ny * nz * 608 / ms / 1e6}

    if a.ab:
        ks = [int(v) for v in a.ab.split(",")]
        tot = {k: 0.0 for k in ks}
        L.step(5)
        for r in range(a.rounds):
            for k in (ks if r % 2 == 0 else ks[::-1]):
                lb.lb_debug_step_kernel(L.h, k)
                L.step(2)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                L.step(a.steps)
                e1.record(stream)
                torch.cuda.synchronize()
                tot[k] += e0.elapsed_time(e1)
        for k in ks:
            out[f"ab_kernel{k}"] = {"mlups": nx * ny * nz * a.steps * a.rounds / tot[k] / 1e3}
        lb.lb_debug_step_kernel(L.h, 0)
        L.close()
        print(json.dumps(out))
        return
    out["step"] = timed(lambda n: L.step(n), "step")
    for name, which in (("step_ws", 3), ("step_tile", 1)):
        try:
            lb.lb_debug_step_kernel(L.h, which)
            out[name] = timed(lambda n: L.step(n), name)
        except lb.LBError as e:
            out[name] = str(e)
    lb.lb_debug_step_kernel(L.h, 0)
    out["probe1_copy_push"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 1), "probe1_copy_push")
    out["probe2_plus_halo_phi_P"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 2), "probe2_plus_halo_phi_P")
    out["probe3_tile_only"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 3), "probe3_tile_only")
    out["probe4_box_no_gtile"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 4), "probe4_box_no_gtile")
    out["probe5_gtile_ahead_ring"] = timed(lambda n: lb.lb_debug_step_probe(L.h, n, 5), "probe5_gtile_ahead_ring")
    out["k_stream_site_parallel"] = timed(lambda n: lb.lb_debug_stream(L.h, n), "k_stream_site_parallel")
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
