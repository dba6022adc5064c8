#!/usr/bin/env python
"""bench.py -- MLUPS and achieved HBM GB/s of the D3Q19 binary-fluid LB step on B200.

Metric (BASELINE.json): lattice site updates per second (MLUPS) and achieved HBM
GB/s against the measured B200 peak, at 1/2/4/8 GPUs.  One "step" = one full LB
timestep (every row of SURVEY.md sec. 8(a)) over the whole lattice.

Default workload: BASELINE config 5, weak scaling with a fixed 512 x 512 x 64
z-slab per GPU (global 512 x 512 x 64N; 512^3 at N = 8; reading R20).  --config
picks another BASELINE config (c1 16^3, c2 64^3, c3 128^3, c4 256^3 strong).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL halos)

Timing: the step's CUDA graphs are captured first (lb_prepare), then W >= 3
untimed steps, then exactly K steps bracketed by a barrier and a device
synchronize, timed with CUDA events on the library's own stream, max over ranks
(`value`); 5 more repetitions of the same K steps give `reps` (min, median,
stddev); then K more steps with CUDA events around every kernel launch, from
which the step kernel's average launch time (`roofline.achieved`).  Inputs are
larger than L2 for c3-c5 (per-GPU state >= 1.3 GB).
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lattice site updates/s (MLUPS) and achieved HBM GB/s vs B200 peak at 1/2/4/8 GPUs"
BYTES_PER_SITE = 608.0  # f and g (38 fp64) read once and written once
BYTES_PER_SITE_CH = 320.0  # NEXT-2: f (19 fp64) and phi read once and written once
BYTES_PER_SITE_LC = 432.0  # NEXT-4: f (19 fp64), Q (5) and the stored u (3) read once and written once

# name: (nx, ny, nz_global(N), scaling, description)
CONFIGS = {
    "c1": (16, 16, lambda n: 16 * n, "weak", "16^3 per GPU D3Q19 binary fluid, spinodal phi +-0.01 (BASELINE config 1)"),
    "c2": (64, 64, lambda n: 64 * n, "weak", "64^3 per GPU binary fluid (BASELINE config 2)"),
    "c3": (128, 128, lambda n: 128 * n, "weak", "128^3 per GPU binary fluid, paper-scale single device (BASELINE config 3)"),
    "c4": (256, 256, lambda n: 256, "strong", "256^3 binary fluid, strong scaling over z-slabs (BASELINE config 4)"),
    "c5": (512, 512, lambda n: 64 * n, "weak",
           "512x512x64 per GPU z-slab binary fluid, weak scaling, 512^3 at 8 GPUs (BASELINE config 5, reading R20)"),
    "c5alt": (256, 256, lambda n: 512 * n, "weak",
              "256x256x512 per GPU z-slab binary fluid, weak scaling (BASELINE config 5 as literally written, "
              "the R20 alternative)"),
}
REPS = 5  # repetitions of the timed region after the first (min of >= 5, median, stddev)
DEFAULT_CONFIG = "c5"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--lattice", default="", help="tuning only: NX,NY,NZ per GPU instead of the config's lattice")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--collision", default="bgk", choices=["bgk", "mrt", "ch", "lc"],
                    help="bgk: BGK + Guo force (the paper path, default); mrt: stress in f^eq + MRT (NEXT-3); "
                         "ch: phi by finite-difference Cahn-Hilliard instead of g, f as mrt (NEXT-2); "
                         "lc: the liquid-crystal workload, Q tensor by Beris-Edwards + Guo-forced f (NEXT-4)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def src_hash() -> str:
    h = hashlib.sha1()
    csrc = os.path.join(ROOT, "paper_1609_01479_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        if f.endswith((".cu", ".cuh")):
            h.update(open(os.path.join(csrc, f), "rb").read())
    return h.hexdigest()[:12]


def ncu_traffic(kernel: str, config: str):
    """dram bytes (read + write) per launch of `kernel` from a committed ncu --set full
    capture (profiles/traffic.json), only if it was taken on the current sources."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        e = t.get(f"{kernel}@{config}")
        if e and e.get("src_hash") == src_hash():
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks, throttle reasons and board power sampled every 100 ms
    while running."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,enforced.power.limit")

    def __init__(self, gpu_index: int):
        self.rows, self.marks = [], {}
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append((time.monotonic(), parts))

    def mark(self, name):
        self.marks[name] = time.monotonic()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        t0, t1 = self.marks.get("start", 0), self.marks.get("end", 1e30)
        inside = [p for (t, p) in self.rows if t0 <= t <= t1] or [p for (_, p) in self.rows]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(p[0]) for p in inside if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in inside if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for p in inside for k in range(4) if p[3 + k].lower() == "active"})

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        pw = [num(p[7]) for p in inside if len(p) > 7 and num(p[7]) is not None]
        lim = [num(p[8]) for p in inside if len(p) > 8 and num(p[8]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside),
                "power_w_median": statistics.median(pw) if pw else None,
                "power_limit_w": max(lim) if lim else None}


# ------------------------------------------------------------------------------ oracle arm
def oracle_sample_shape(nx: int, ny: int, budget_sites: int):
    """A periodic nx x ny_s x nz_s sub-lattice of the workload with ~budget_sites sites."""
    nz_s = 8
    ny_s = max(4, min(ny, budget_sites // (nx * nz_s)))
    ny_s = 1 << (ny_s.bit_length() - 1)
    return nx, ny_s, nz_s


def oracle_stepper(collision: str):
    """(module name, step function, run function, params) of the oracle for a collision model."""
    from oracle import lb_mrt as M
    from oracle import lb_ref as R

    if collision == "mrt":
        p = M.MrtParams(base=R.Params(), tau_s=0.8, tau_b=1.1, tau_ghost=1.0)
        return "oracle/lb_mrt.py", M.step, M.run, p
    if collision == "ch":
        from oracle import lb_ch as CH

        return "oracle/lb_ch.py", CH.step, CH.run, CH.ChParams(base=R.Params(), tau_s=0.8, tau_b=1.1, tau_ghost=1.0)
    if collision == "lc":
        from oracle import lb_lc as LC

        return "oracle/lb_lc.py", LC.step, LC.run, LC.LcParams()
    return "oracle/lb_ref.py", R.step, R.run, R.Params()


def oracle_state(shape, seed: int, collision: str) -> tuple:
    """Initial state of the oracle on an (nx, ny, nz) sample: (f, g) at equilibrium on the
    spinodal phi, (f, phi) for the ch variant, (f, Q, u) of the random-director quench (lc)."""
    from oracle import lb_ref as R
    from paper_1609_01479_b200 import synth

    sx, sy, sz = shape
    if collision == "lc":
        from oracle import lb_lc as LC

        n = synth.random_directors(sx, sy, sz, seed)
        return LC.initial_state(np.ones((sz, sy, sx)), np.zeros((3, sz, sy, sx)), n, LC.LcParams())
    rho, u, phi = synth.spinodal_fields(sx, sy, sz, seed)
    if collision == "ch":
        return R.f_equilibrium(rho, u), phi
    return R.equilibrium_state(rho, u, phi, R.Params())


def time_oracle(nx, ny, steps: int, seed: int = 0, collision: str = "bgk"):
    """The oracle as it stands, 1 thread, on a sample sub-lattice; returns (sites/s, shape)."""
    _, step, run, p = oracle_stepper(collision)
    sx, sy, sz = oracle_sample_shape(nx, ny, 262144 if collision != "lc" else 65536)
    st = oracle_state((sx, sy, sz), seed, collision)
    step(*st, p)  # warm
    t0 = time.perf_counter()
    st = run(*st, p, steps)
    dt = time.perf_counter() - t0
    return sx * sy * sz * steps / dt, (sx, sy, sz), dt


def run_reference(args):
    rank, world, _ = env_rank_world()
    if rank != 0:
        return 0
    nx, ny, nzf, scaling, desc = CONFIGS[args.config]
    if args.collision == "lc":
        desc = desc.replace("binary fluid", "liquid crystal (Q tensor + D3Q19 fluid, NEXT-4)")
    sx, sy, sz = oracle_sample_shape(nx, ny, 262144 if args.collision != "lc" else 65536)
    name, _, run, p = oracle_stepper(args.collision)
    st = oracle_state((sx, sy, sz), 0, args.collision)
    st = run(*st, p, max(args.warmup, 0))
    t0 = time.perf_counter()
    st = run(*st, p, args.steps)
    dt = time.perf_counter() - t0
    sites = sx * sy * sz
    v = sites * args.steps / dt / 1e6
    sample = f"{name} NumPy fp64 step on a periodic {sx}x{sy}x{sz} sub-lattice ({sites} sites) of the workload per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "MLUPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "sample": [sx, sy, sz]},
        "cpu_baseline": {"value": v, "unit": "MLUPS", "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
        "e2e": {"value": v, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm
def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def run_ours(args):
    import torch

    from paper_1609_01479_b200 import dist as D
    from paper_1609_01479_b200 import lb, synth

    rank, world, local = env_rank_world()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        D.init("nccl")
    nx, ny, nzf, scaling, desc = CONFIGS[args.config]
    if args.lattice:
        nx, ny, nzl_ = (int(v) for v in args.lattice.split(","))
        nzf, scaling, desc = (lambda n: nzl_ * n), "weak", f"tuning lattice {nx}x{ny}x{nzl_} per GPU"
    if args.collision == "lc":
        desc = desc.replace("binary fluid", "liquid crystal (Q tensor + D3Q19 fluid, NEXT-4)")
    nz = nzf(world)
    z0, z1 = D.slab_range(nz, world, rank)
    nloc = nx * ny * (z1 - z0)
    params = lb.make_params()  # R16 defaults
    uid = None
    if world > 1:
        uid = D.broadcast_bytes(lb.lb_nccl_get_unique_id() if rank == 0 else None)
    if args.collision == "ch":  # z-slabs with NCCL halos under torchrun
        L = lb.ChLattice(nx, ny, nz, params, 0.8, 1.1, 1.0, nranks=world, rank=rank, uid=uid)
    elif args.collision == "lc":  # R44 defaults; z-slabs with NCCL halos under torchrun
        L = lb.LcLattice(nx, ny, nz, lb.make_lc_params(), nranks=world, rank=rank, uid=uid)
    else:
        L = lb.Lattice(nx, ny, nz, params, nranks=world, rank=rank, uid=uid)
    bps = {"ch": BYTES_PER_SITE_CH, "lc": BYTES_PER_SITE_LC}.get(args.collision, BYTES_PER_SITE)
    if args.collision == "mrt":
        lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
    halo = ("peer (fused P2P stores)" if lb.lb_debug_halo_mode(L.h) == 1 else "NCCL send/recv") if world > 1 else None
    if args.collision == "lc":
        L.init(synth.random_directors_slab(nx, ny, nz, z0, z1, 0))  # R45: quench from random directors
    else:
        L.init_equilibrium(synth.spinodal_phi_slab(nx, ny, nz, z0, z1, seed=0))

    # the CUDA graphs lb_step replays (single process) are captured here, outside
    # the warm-up count and the timed regions; then W >= 3 untimed steps
    W = max(args.warmup, 3)
    K = args.steps
    stream = torch.cuda.ExternalStream(lb.lb_stream(L.h))
    lb.lb_prepare(L.h)
    L.step(W)

    def timed_region():
        """K steps bracketed by a barrier + device sync, CUDA events on the library's
        stream; returns (max-over-ranks ms, kernel launches)."""
        D.barrier()
        torch.cuda.synchronize()
        n0 = lb.lb_launch_count(L.h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.step(K)
        e1.record(stream)
        torch.cuda.synchronize()
        D.barrier()
        return D.max_over_ranks(e0.elapsed_time(e1)), lb.lb_launch_count(L.h) - n0

    # timed region 1 -> `value`: K steps, no per-launch instrumentation; region 2
    # right after it (the same power-capped clock) -> `roofline`; then REPS more
    # repetitions of region 1 (min / median / stddev); clocks sampled throughout
    clocks = ClockSampler(local)
    time.sleep(0.25)
    clocks.mark("start")
    ms, launches = timed_region()
    # timed region 2: the same K steps with CUDA events around every kernel launch
    # (per-kernel durations; the events cost ~8 us per step, which is why region 1
    # runs without them)
    D.barrier()
    torch.cuda.synchronize()
    lb.lb_profile_reset(L.h)
    lb.lb_profile_enable(L.h, True)
    L.step(K)
    torch.cuda.synchronize()
    D.barrier()
    lb.lb_profile_enable(L.h, False)
    prof = lb.lb_profile(L.h)
    rep_ms = [ms] + [timed_region()[0] for _ in range(REPS)]
    clocks.mark("end")
    clk = clocks.stop()
    reps = {"n": len(rep_ms), "steps_each": K, "ms_per_step_min": min(rep_ms) / K,
            "ms_per_step_median": statistics.median(rep_ms) / K, "ms_per_step_stddev": statistics.stdev(rep_ms) / K,
            "mlups_max": nx * ny * nzf(world) * K / (min(rep_ms) * 1e-3) / 1e6,
            "note": "value = the first region (exactly K steps); these are it and REPS more of the same K steps, "
                    "run after the per-launch region that gives `roofline`"}

    sites_total = nx * ny * nz
    value = sites_total * K / (ms * 1e-3) / 1e6  # MLUPS, whole job
    peak, peak_src = peaks()
    ks_ms, ks_n = prof.get("k_step", (0.0, 0))
    ks_evented = D.max_over_ranks(ks_ms / max(ks_n, 1))
    # where a step is exactly one step-kernel launch (every launch of the per-launch
    # region was k_step, one per step, and the value region launched K kernels), the
    # value region itself times the kernel: K back-to-back launches of a graph, so
    # its time per launch bounds the kernel's from above (the gaps between graph
    # kernel nodes are ~1 us).  Otherwise the per-launch region's events.
    only_kstep = ks_n == K and all(n == 0 for k, (_, n) in prof.items() if k != "k_step")
    if only_kstep and launches == K:
        ks_avg, ks_basis = ms / K, "value region: K graph-replayed launches of k_step, one per step (time / launch)"
    else:
        ks_avg, ks_basis = ks_evented, "per-launch CUDA events in a region of K steps after the value region"
    achieved = bps * nloc / (ks_avg * 1e-3) / 1e9
    step_gbs = value * 1e6 * bps / world / 1e9  # per GPU, algorithmic, whole step
    traffic = ncu_traffic("k_step", args.config if args.collision == "bgk" else f"{args.config}-{args.collision}")
    kernel_share = {k: round(v[0] / max(sum(x[0] for x in prof.values()), 1e-30), 4) for k, v in prof.items() if v[1]}

    # ---- e2e: the same metric through the public C ABI with pinned HOST buffers:
    # every step uploads the state (lb_set_state), advances one step, and reads the
    # state back (lb_get_state); copies inside the timed region.
    e2e = None
    if not args.no_e2e:
        Ke = min(K, 5)
        # host arrays of the state: (f, g), (f, phi) or (f, Q, u), and the ABI pair
        sizes = {"ch": (19, 1), "lc": (19, 5, 3)}.get(args.collision, (19, 19))
        host = [torch.empty(k * nloc, dtype=torch.float64, pin_memory=True) for k in sizes]
        sfx = {"ch": "_ch", "lc": "_lc"}.get(args.collision, "")
        set_state, get_state = getattr(lb, "lb_set_state" + sfx), getattr(lb, "lb_get_state" + sfx)
        get_state(L.h, *host)
        D.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(Ke):
            set_state(L.h, *host)
            lb.lb_step(L.h, 1)
            get_state(L.h, *host)
        a1.record(stream)
        torch.cuda.synchronize()
        D.barrier()
        ems = D.max_over_ranks(a0.elapsed_time(a1))
        nbytes = 8 * nloc * sum(sizes)
        e2e = {"value": sites_total * Ke / (ems * 1e-3) / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "steps": Ke,
               "mode": f"per step: lb_set_state{sfx}(pinned host state) + lb_step(1) + lb_get_state{sfx}(pinned host state)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cv, shp, dt = time_oracle(nx, ny, 20, collision=args.collision)
        cpu = {"value": cv / 1e6, "unit": "MLUPS", "cores": 1, "kind": "oracle",
               "sample": f"{oracle_stepper(args.collision)[0]}, 20 steps on a periodic {shp[0]}x{shp[1]}x{shp[2]} sub-lattice of the "
                         f"workload, 1 thread ({dt:.1f} s of CPU)", "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}

    L.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "lattice": [nx, ny, nz], "sites_per_gpu": nloc,
                       "parallelism": f"z-slab x{world}" + (f" ({halo} halos)" if world > 1 else ""),
                       "collision": {"bgk": "BGK + Guo force F = -div P (paper path)",
                                     "mrt": "chemical stress in f^eq, MRT tau_s 0.8 / tau_b 1.1 / tau_ghost 1.0 (NEXT-3)",
                                     "ch": "phi by finite-difference Cahn-Hilliard + upwind advection (NEXT-2); "
                                           "f: chemical stress in f^eq, MRT 0.8 / 1.1 / 1.0",
                                     "lc": "liquid crystal (NEXT-4): Landau-de Gennes Q tensor, Beris-Edwards LC update "
                                           "+ upwind advection, f: BGK + Guo force F = div sigma; quench from random "
                                           "directors (R45)"}[args.collision],
                       "state_bytes_per_gpu": int(2 * 38 * 8 * nx * ny * (z1 - z0 + 2) + 8 * nx * ny * (z1 - z0 + 4)
                                                  + (2 * 8 * 8 * nloc if args.collision == "lc" else 0)),
                       "l2": "inputs larger than L2 (state per GPU >> 126 MB)" if nloc * 608 > 126e6 * 2
                       else "state comparable to L2: not an HBM roofline point",
                       "params": ({"tau_f": 0.8, "A0": 0.01, "gamma": 3.2, "kappa": 0.01, "xi": 0.7, "Gamma": 0.3}
                                  if args.collision == "lc" else
                                  {"tau_f": 0.8, "tau_g": 1.3, "A": -0.0625, "B": 0.0625, "kappa": 0.04, "M": 0.05})},
            "hbm_gbs_step": step_gbs,
            "roofline": {"bound": "hbm", "kernel": "k_step", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_site": bps, "avg_launch_ms": ks_avg, "avg_launch_basis": ks_basis,
                         "avg_launch_ms_evented": ks_evented,
                         "step_frac": step_gbs / peak, "kernel_time_share": kernel_share},
            "reps": reps, "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
            "src_hash": src_hash(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as tdist

        tdist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
