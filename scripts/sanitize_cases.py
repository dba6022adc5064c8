"""Small cases of every step kernel, checked for memory safety without
compute-sanitizer (closed on this pool): after each run the guard zones around
every field buffer must be intact (lb_debug_guards == 0) and, with the
bounds-checked build (LB_VARIANT=checked), no device index check may have failed
(lb_debug_check == 0); buffers start NaN-filled, so a read of memory nobody wrote
shows up as an oracle mismatch.  Cases:
the warp-specialised kernel with the phi exchange (16^3 default), the plain
warp-specialised and tile kernels, 32 x 8 tiles over several waves with a
wrapped box, two loopback slabs with the peer transport (K_phi edges, P2P
pushes, device-side epochs), the MRT collision, the Cahn-Hilliard and the
liquid-crystal kernels.  Exits non-zero if any result misses the oracle or any
check fails.

  LB_VARIANT=checked python scripts/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import lb_ch as CH  # noqa: E402
from oracle import lb_lc as LC  # noqa: E402
from oracle import lb_mrt as M  # noqa: E402
from oracle import lb_ref as R  # noqa: E402
from paper_1609_01479_b200 import lb, synth  # noqa: E402

P = R.Params()
CP = lb.make_params(P.tau_f, P.tau_g, P.A, P.B, P.kappa, P.mobility)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def rough(nx, ny, nz, seed=1):
    rho, u, phi, nf, ng = synth.rough_fields(nx, ny, nz, seed)
    f, g = R.equilibrium_state(rho, u, phi, P)
    return f + nf, g + ng


bad = []


def memsafe(L, name):
    guards = lb.lb_debug_guards(L.h)
    line = lb.lb_debug_check(L.h)
    print(f"  {name}: guard bytes changed {guards}, failed device check at line {line}", flush=True)
    if guards or line:
        bad.append(name + " (memory)")


print("bounds-checked build:", lb.lb_debug_checked(), flush=True)
for (shape, kernel, nslabs, halo, steps) in [((16, 16, 16), 0, 1, None, 3), ((16, 16, 16), 2, 1, None, 2),
                                             ((17, 12, 8), 1, 1, None, 2), ((64, 24, 6), 2, 1, None, 1), ((96, 41, 6), 2, 1, None, 1),
                                             ((32, 16, 8), 0, 2, 1, 2), ((32, 16, 8), 1, 2, 1, 2),
                                             ((32, 16, 8), 0, 2, 0, 2)]:
    nx, ny, nz = shape
    f, g = rough(nx, ny, nz)
    with lb.Lattice(nx, ny, nz, CP, nslabs=nslabs) as L:
        lb.lb_debug_step_kernel(L.h, kernel)
        if halo is not None:
            lb.lb_debug_halo_mode(L.h, halo)
        L.set_state(f, g)
        L.step(steps)
        f1, g1 = L.get_state()
        memsafe(L, f"{shape} kernel {kernel} slabs {nslabs}")
    f0, g0 = R.run(f, g, P, steps)
    e = max(rel(f1, f0), rel(g1, g0))
    print(f"case {shape} kernel {kernel} slabs {nslabs} halo {halo}: rel err {e:.2e}", flush=True)
    if not e <= 1e-12:
        bad.append(shape)

# MRT collision (NEXT-3)
mp = M.MrtParams(base=P, tau_s=0.8, tau_b=1.1, tau_ghost=1.0)
f, g = rough(16, 8, 8)
with lb.Lattice(16, 8, 8, CP) as L:
    lb.lb_set_collision(L.h, 1, 0.8, 1.1, 1.0)
    L.set_state(f, g)
    L.step(2)
    f1, g1 = L.get_state()
    memsafe(L, "mrt")
f0, g0 = M.run(f, g, mp, 2)
e = max(rel(f1, f0), rel(g1, g0))
print(f"case mrt: rel err {e:.2e}", flush=True)
bad += [] if e <= 1e-12 else ["mrt"]

# Cahn-Hilliard (NEXT-2)
rho, u, phi = synth.spinodal_fields(16, 8, 8, 0)
fch = R.f_equilibrium(rho, u)
with lb.ChLattice(16, 8, 8, CP, 0.8, 1.1, 1.0) as L:
    L.set_state(fch, phi)
    L.step(2)
    f1, p1 = L.get_state()
    memsafe(L, "ch")
f0, p0 = CH.run(fch, phi, CH.ChParams(base=P, tau_s=0.8, tau_b=1.1, tau_ghost=1.0), 2)
e = max(rel(f1, f0), rel(p1, p0))
print(f"case ch: rel err {e:.2e}", flush=True)
bad += [] if e <= 1e-12 else ["ch"]

# liquid crystal (NEXT-4)
lp = LC.LcParams()
st = LC.initial_state(rho, u, synth.random_directors(16, 8, 8, 0), lp)
with lb.LcLattice(16, 8, 8, lb.make_lc_params(lp.tau_f, lp.A0, lp.gamma, lp.kappa, lp.xi, lp.Gamma)) as L:
    L.set_state(*st)
    L.step(2)
    got = L.get_state()
    memsafe(L, "lc")
ref = LC.run(*st, lp, 2)
e = max(rel(got[0], ref[0]), rel(got[1], ref[1]))
print(f"case lc: rel err {e:.2e}", flush=True)
bad += [] if e <= 1e-12 else ["lc"]

print("sanitize cases:", "FAILED " + str(bad) if bad else "all ok")
sys.exit(1 if bad else 0)
