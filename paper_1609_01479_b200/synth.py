"""Seeded synthetic inputs shared by the tests, the oracle leg and the bench.

This module holds random numbers and array shapes only -- none of the
method's arithmetic (no moments, stencils or equilibria).  Both the CUDA path
(through the C ABI) and the CPU oracle are fed from here; everything else
about the initial state is computed by each side on its own (the GPU by
``lb_init_equilibrium``, the oracle by ``oracle.lb_ref.equilibrium_state``).

Recipe (BASELINE.json configs; reading R15):
  spinodal   phi = phi0 + amp * (2U - 1), U ~ U[0,1) i.i.d. from NumPy's
             PCG64 ``default_rng(seed)``, drawn in canonical site order
             s = x + nx*(y + ny*z); rho = 1, u = 0.
  rough      phi ~ U(-0.8, 0.8), rho = 1 + 0.05 U, |u_a| <= 0.02, plus noise
             arrays of amplitude 1e-3 for f and g (exercises every term).
All arrays are float64, shaped (nz, ny, nx) or (k, nz, ny, nx).
"""
from __future__ import annotations

import numpy as np

Q = 19  # number of distribution components per site (D3Q19)


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def spinodal_phi(nx: int, ny: int, nz: int, seed: int = 0, phi0: float = 0.0, amp: float = 0.01) -> np.ndarray:
    """Order parameter of a quench into the spinodal region: phi0 +- amp noise."""
    u = _rng(seed).random(nx * ny * nz)
    return (phi0 + amp * (2.0 * u - 1.0)).reshape(nz, ny, nx)


def spinodal_phi_slab(nx: int, ny: int, nz: int, z0: int, z1: int, seed: int = 0, phi0: float = 0.0,
                      amp: float = 0.01) -> np.ndarray:
    """Planes [z0, z1) of ``spinodal_phi(nx, ny, nz, seed)``, bitwise, without drawing
    the rest: the PCG64 stream is advanced past the z0*nx*ny earlier sites."""
    del nz  # the global extent does not change the draws of these planes
    bg = np.random.PCG64(seed)
    bg.advance(z0 * nx * ny)
    u = np.random.Generator(bg).random(nx * ny * (z1 - z0))
    return (phi0 + amp * (2.0 * u - 1.0)).reshape(z1 - z0, ny, nx)


def spinodal_fields(nx: int, ny: int, nz: int, seed: int = 0, phi0: float = 0.0, amp: float = 0.01):
    """(rho, u, phi) of the spinodal initial state: rho = 1, u = 0."""
    rho = np.ones((nz, ny, nx))
    u = np.zeros((3, nz, ny, nx))
    return rho, u, spinodal_phi(nx, ny, nz, seed, phi0, amp)


def rough_fields(nx: int, ny: int, nz: int, seed: int = 1):
    """(rho, u, phi, noise_f, noise_g): a rough state that exercises every term."""
    r = _rng(seed)
    shape = (nz, ny, nx)
    phi = r.uniform(-0.8, 0.8, size=shape)
    rho = 1.0 + 0.05 * r.random(shape)
    u = r.uniform(-0.02, 0.02, size=(3,) + shape)
    noise_f = 1e-3 * r.uniform(-1.0, 1.0, size=(Q,) + shape)
    noise_g = 1e-3 * r.uniform(-1.0, 1.0, size=(Q,) + shape)
    return rho, u, phi, noise_f, noise_g


def sample_sites(nx: int, ny: int, nz: int, n: int, seed: int = 7) -> list[tuple[int, int, int]]:
    """n distinct sampled sites, always including the 8 corners (wrap-around edges)."""
    r = _rng(seed)
    corners = [(x, y, z) for x in (0, nx - 1) for y in (0, ny - 1) for z in (0, nz - 1)]
    picks = set(corners)
    while len(picks) < min(n, nx * ny * nz):
        picks.add((int(r.integers(nx)), int(r.integers(ny)), int(r.integers(nz))))
    return sorted(picks, key=lambda s: (s[2], s[1], s[0]))


# ---- NEXT-4 liquid-crystal workload (R45) ------------------------
def random_directors(nx: int, ny: int, nz: int, seed: int = 0) -> np.ndarray:
    """Unit vectors n (3, nz, ny, nx), uniform on the sphere: per site (canonical site
    order) two uniforms U1, U2 of PCG64 ``default_rng(seed)``, cos(theta) = 2 U1 - 1,
    phi = 2 pi U2."""
    return random_directors_slab(nx, ny, nz, 0, nz, seed)


def random_directors_slab(nx: int, ny: int, nz: int, z0: int, z1: int, seed: int = 0) -> np.ndarray:
    """Planes [z0, z1) of ``random_directors(nx, ny, nz, seed)``, bitwise, without drawing
    the rest (the stream is advanced past the 2 z0 nx ny earlier draws)."""
    del nz
    bg = np.random.PCG64(seed)
    bg.advance(2 * z0 * nx * ny)
    uv = np.random.Generator(bg).random(2 * nx * ny * (z1 - z0)).reshape(-1, 2)
    c = 2.0 * uv[:, 0] - 1.0
    s = np.sqrt(1.0 - c * c)
    ph = 2.0 * np.pi * uv[:, 1]
    return np.stack([s * np.cos(ph), s * np.sin(ph), c]).reshape(3, z1 - z0, ny, nx)


def rough_lc_fields(nx: int, ny: int, nz: int, seed: int = 3):
    """(rho, u, q5, noise_f): a rough liquid-crystal state that exercises every term:
    the five stored Q components ~ U(-0.3, 0.3), rho = 1 + 0.05 U, |u_a| <= 0.02,
    f noise of amplitude 1e-3."""
    r = _rng(seed)
    shape = (nz, ny, nx)
    q5 = r.uniform(-0.3, 0.3, size=(5,) + shape)
    rho = 1.0 + 0.05 * r.random(shape)
    u = r.uniform(-0.02, 0.02, size=(3,) + shape)
    noise_f = 1e-3 * r.uniform(-1.0, 1.0, size=(Q,) + shape)
    return rho, u, q5, noise_f
