"""Schedule of the warp-specialised step kernel's blocks (a measurement build:
LB_NVCC_FLAGS=-DLB_TRACE, loaded as LB_VARIANT=trace): per block start / end
time and SM; prints, per setting, the block durations and the time between a
tile and its x / y neighbours reaching the same plane (in plane-times).
  LB_VARIANT=trace python scripts/trace_schedule.py NX NY NZ "zc=0" "zc=16" "band=2" ...
(always the halo-box kernel, lb_debug_step_kernel 2)"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401

from paper_1609_01479_b200 import lb, synth  # noqa: E402

KEYS = {"zc": lb.LB_TUNE_ZCHUNK, "band": lb.LB_TUNE_BAND_ROWS, "resid": lb.LB_TUNE_RESID}
DEFAULTS = {"zc": 0, "band": 1, "resid": 0}
nx, ny, nz = (int(v) for v in sys.argv[1:4])
res = {}
with lb.Lattice(nx, ny, nz) as L:
    lib = lb._lib
    lib.lb_debug_trace_get.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lb.lb_debug_tune(L.h, lb.LB_TUNE_GRAPHS, 0)
    lb.lb_debug_step_kernel(L.h, 2)
    L.init_equilibrium(synth.spinodal_phi(nx, ny, nz, seed=0))
    L.step(3)
    torch.cuda.synchronize()
    lib.lb_debug_trace_get(np.zeros((1 << 16, 4), dtype=np.uint64).ctypes.data, 1 << 16)  # clear
    for s in sys.argv[4:]:
        for kv in s.split(","):
            k, v = kv.split("=")
            lb.lb_debug_tune(L.h, KEYS[k], int(v))
        L.step(1)
        torch.cuda.synchronize()
        nb = 1 << 16
        buf = np.zeros((nb, 4), dtype=np.uint64)
        assert lib.lb_debug_trace_get(buf.ctypes.data, nb) == 0
        used = buf[:, 1] > 0
        b = buf[used]
        t0 = b[:, 0].astype(np.int64)
        t1 = b[:, 1].astype(np.int64)
        tmin = t0.min()
        t0 -= tmin
        t1 -= tmin
        bx = (b[:, 3] >> 40).astype(np.int64)
        by = ((b[:, 3] >> 20) & 0xFFFFF).astype(np.int64)
        zA = (b[:, 3] & 0xFFFFF).astype(np.int64)
        zb_ = (b[:, 2] >> 32).astype(np.int64)
        dur = (t1 - t0)
        n = len(b)
        zc = int(np.round(np.mean(zb_ - zA)))  # planes per block (mean)
        pt = (dur / (zb_ - zA)).mean()  # one plane-time, ns
        # time each (tile, plane) is processed
        ntx, nty = nx // 32, ny // 8
        T = np.full((nty, ntx, nz), np.nan)
        for i in range(n):
            m = zb_[i] - zA[i]
            for j in range(m):
                p = (zA[i] + j) % nz
                T[by[i], bx[i], p] = t0[i] + (j + 0.5) * dur[i] / m
        dy = np.abs(T - np.roll(T, -1, axis=0)) / pt
        dx = np.abs(T - np.roll(T, -1, axis=1)) / pt
        q = lambda a: [round(float(np.nanpercentile(a, v)), 2) for v in (10, 50, 90, 99)]
        res[s] = {"blocks": n, "zc": zc, "plane_time_us": round(pt / 1e3, 3), "kernel_us": round((t1.max()) / 1e3, 1),
                  "dur_us_p10_50_90": [round(float(np.percentile(dur, v)) / 1e3, 1) for v in (10, 50, 90)],
                  "y_lag_planes_p10_50_90_99": q(dy), "x_lag_planes_p10_50_90_99": q(dx),
                  "start_spread_first_wave_us": round(float(np.sort(t0)[:148].max()) / 1e3, 2)}
        sm = (b[:, 2] & 0xFFFFFFFF).astype(np.int64)
        nsm = int(sm.max()) + 1
        sm_end = np.array([t1[sm == i].max() for i in range(nsm) if (sm == i).any()])
        sm_busy = np.array([dur[sm == i].sum() for i in range(nsm) if (sm == i).any()])
        res[s].update({"sms": len(sm_end), "busy_fraction": round(float(dur.sum() / (len(sm_end) * t1.max())), 4),
                       "sm_end_us_min_p50_max": [round(float(v) / 1e3, 1) for v in (sm_end.min(), np.median(sm_end),
                                                                                      sm_end.max())],
                       "sm_busy_us_min_p50_max": [round(float(v) / 1e3, 1) for v in (sm_busy.min(), np.median(sm_busy),
                                                                                       sm_busy.max())],
                       "last_start_us": round(float(t0.max()) / 1e3, 1)})
        # duration by tile class: the box wraps (cp.async) or not (TMA)
        edge = (bx == 0) | (bx == ntx - 1) | (by == 0) | (by == nty - 1)
        res[s]["dur_us_interior_edge"] = [round(float(dur[~edge].mean()) / 1e3, 1),
                                          round(float(dur[edge].mean()) / 1e3, 1) if edge.any() else None]
        for kv in s.split(","):
            k, _ = kv.split("=")
            lb.lb_debug_tune(L.h, KEYS[k], DEFAULTS[k])
print(json.dumps(res, indent=1))
