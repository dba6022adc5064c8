"""Brute-force scalar oracle: per-site Python loops over Python floats (fp64).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.

A second, deliberately naive transcription of the same step as ``lb_ref``
(readings R1-R14 of DESIGN.md; PAPER.md P:163-190 for the components, S:331-348
for the BGK/propagation forms).  It shares no tables or formulas with
``lb_ref``: the velocity set is *enumerated* here (all c in {-1,0,1}^3 with
|c|^2 <= 2, rest first, then descending lexicographic (cx, cy, cz)) instead of
typed in, and every sum is an explicit loop over sites and components.  It is
used

* on whole lattices of at most ~8^3 sites (``step``), to cross-check ``lb_ref``;
* on single sampled sites of lattices of any size (``site_after_step``), to
  check the GPU path at full benchmark sizes where ``lb_ref`` would be slow.

Arguments ``p`` may be any object with attributes tau_f, tau_g, A, B, kappa,
mobility.
"""
from __future__ import annotations

import itertools

import numpy as np


def velocity_set() -> tuple[list[tuple[int, int, int]], list[float]]:
    """R1 by enumeration: D3Q19 = {c in {-1,0,1}^3 : |c|^2 <= 2}; order of Appendix B."""
    cs = [c for c in itertools.product((1, 0, -1), repeat=3) if sum(v * v for v in c) <= 2]
    cs.remove((0, 0, 0))
    cs.sort(reverse=True)  # descending lexicographic (cx, cy, cz)
    cs.insert(0, (0, 0, 0))
    w = [{0: 1.0 / 3.0, 1: 1.0 / 18.0, 2: 1.0 / 36.0}[sum(v * v for v in c)] for c in cs]
    return cs, w


CV, WV = velocity_set()
Q = len(CV)


class _Site:
    """Periodic scalar access to one state (Python lists, x fastest)."""

    def __init__(self, f: np.ndarray, g: np.ndarray, p):
        self.q, self.nz, self.ny, self.nx = f.shape
        self.f = f.tolist()
        self.g = g.tolist()
        self.p = p
        self._phi: dict = {}
        self._P: dict = {}

    def wrap(self, x, y, z):
        return x % self.nx, y % self.ny, z % self.nz

    def phi(self, x, y, z):
        """phi = sum_i g_i (A.3)."""
        key = self.wrap(x, y, z)
        if key not in self._phi:
            X, Y, Z = key
            s = 0.0
            for i in range(Q):
                s += self.g[i][Z][Y][X]
            self._phi[key] = s
        return self._phi[key]

    def grad_lap(self, x, y, z):
        """Central gradient and 7-point Laplacian of phi (A.2)."""
        e = ((1, 0, 0), (0, 1, 0), (0, 0, 1))
        grad = []
        lap = 0.0
        for a in range(3):
            up = self.phi(x + e[a][0], y + e[a][1], z + e[a][2])
            dn = self.phi(x - e[a][0], y - e[a][1], z - e[a][2])
            grad.append(0.5 * (up - dn))
            lap += up + dn
        lap -= 6.0 * self.phi(x, y, z)
        return grad, lap

    def mu(self, x, y, z):
        p = self.p
        ph = self.phi(x, y, z)
        _, lap = self.grad_lap(x, y, z)
        return p.A * ph + p.B * ph * ph * ph - p.kappa * lap

    def stress(self, x, y, z):
        """P_ab (A.4) as a 3x3 nested list."""
        key = self.wrap(x, y, z)
        if key not in self._P:
            p = self.p
            ph = self.phi(x, y, z)
            grad, lap = self.grad_lap(x, y, z)
            g2 = grad[0] * grad[0] + grad[1] * grad[1] + grad[2] * grad[2]
            iso = 0.5 * p.A * ph * ph + 0.75 * p.B * ph * ph * ph * ph - p.kappa * ph * lap - 0.5 * p.kappa * g2
            self._P[key] = [[(iso if a == b else 0.0) + p.kappa * grad[a] * grad[b] for b in range(3)] for a in range(3)]
        return self._P[key]

    def force(self, x, y, z):
        """F_a = -sum_b (P_ab(x+e_b) - P_ab(x-e_b))/2 (A.5)."""
        e = ((1, 0, 0), (0, 1, 0), (0, 0, 1))
        F = [0.0, 0.0, 0.0]
        for b in range(3):
            Pu = self.stress(x + e[b][0], y + e[b][1], z + e[b][2])
            Pd = self.stress(x - e[b][0], y - e[b][1], z - e[b][2])
            for a in range(3):
                F[a] -= 0.5 * (Pu[a][b] - Pd[a][b])
        return F

    def collide(self, x, y, z):
        """Post-collision (f*, g*) at one site (A.3-A.7)."""
        p = self.p
        X, Y, Z = self.wrap(x, y, z)
        f = [self.f[i][Z][Y][X] for i in range(Q)]
        g = [self.g[i][Z][Y][X] for i in range(Q)]
        rho = 0.0
        j = [0.0, 0.0, 0.0]
        for i in range(Q):
            rho += f[i]
            for a in range(3):
                j[a] += CV[i][a] * f[i]
        if not (rho > 0.0) or any(v != v or v in (float("inf"), float("-inf")) for v in f + g):
            raise ArithmeticError(f"rho <= 0 or non-finite value at site (x={X}, y={Y}, z={Z})")
        ph = self.phi(X, Y, Z)
        mu = self.mu(X, Y, Z)
        F = self.force(X, Y, Z)
        u = [(j[a] + 0.5 * F[a]) / rho for a in range(3)]
        uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2]
        uF = u[0] * F[0] + u[1] * F[1] + u[2] * F[2]
        gamma = p.mobility / (p.tau_g - 0.5)
        fs, gs = [], []
        for i in range(Q):
            c = CV[i]
            cu = c[0] * u[0] + c[1] * u[1] + c[2] * u[2]
            cF = c[0] * F[0] + c[1] * F[1] + c[2] * F[2]
            c2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2]
            feq = WV[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu)
            S = WV[i] * (3.0 * (cF - uF) + 9.0 * cu * cF)
            fs.append(f[i] - (f[i] - feq) / p.tau_f + (1.0 - 1.0 / (2.0 * p.tau_f)) * S)
            geq = WV[i] * (3.0 * ph * cu + 4.5 * gamma * mu * (c2 - 1.0) + 4.5 * ph * (cu * cu - uu / 3.0))
            if i == 0:
                geq += ph
            gs.append(g[i] - (g[i] - geq) / p.tau_g)
        return fs, gs


def step(f: np.ndarray, g: np.ndarray, p) -> tuple[np.ndarray, np.ndarray]:
    """Whole-lattice step by loops: collide every site, then push f_i*(x) to x + c_i."""
    s = _Site(f, g, p)
    fo = np.empty_like(f)
    go = np.empty_like(g)
    for z in range(s.nz):
        for y in range(s.ny):
            for x in range(s.nx):
                fs, gs = s.collide(x, y, z)
                for i in range(Q):
                    X, Y, Z = s.wrap(x + CV[i][0], y + CV[i][1], z + CV[i][2])
                    fo[i, Z, Y, X] = fs[i]
                    go[i, Z, Y, X] = gs[i]
    return fo, go


class SiteSampler:
    """Post-step values at chosen sites of an arbitrarily large lattice.

    f_i(x, t+1) = f_i*(x - c_i, t): collide the 19 upstream sites, keep the
    component that streams into x.  Caches phi and P across samples.
    """

    def __init__(self, f: np.ndarray, g: np.ndarray, p):
        self.s = _Site(f, g, p)

    def after_step(self, x: int, y: int, z: int) -> tuple[list[float], list[float]]:
        fo, go = [], []
        for i in range(Q):
            fs, gs = self.s.collide(x - CV[i][0], y - CV[i][1], z - CV[i][2])
            fo.append(fs[i])
            go.append(gs[i])
        return fo, go


def propagation_source(nx: int, ny: int, nz: int, x: int, y: int, z: int, i: int) -> tuple[int, int, int]:
    """Integer map: site whose component i streams into (x, y, z) (A.8, periodic)."""
    return (x - CV[i][0]) % nx, (y - CV[i][1]) % ny, (z - CV[i][2]) % nz
