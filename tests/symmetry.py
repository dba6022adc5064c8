"""Cubic point-group action on lattice fields, for the oracle symmetry pins.

Test helper only (no method arithmetic): relabels sites and velocity indices.
"""
import numpy as np

from oracle import lb_ref as R

# reflections in each axis, a transposition, and two axis cycles (one with signs)
CUBIC = [
    np.diag([-1, 1, 1]), np.diag([1, -1, 1]), np.diag([1, 1, -1]),
    np.array([[0, 1, 0], [1, 0, 0], [0, 0, 1]]),
    np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0]]),
    np.array([[0, -1, 0], [0, 0, 1], [-1, 0, 0]]),
]


def cube_transform(a, M, n):
    """Apply the signed permutation M to a periodic n^3 field: a (19, n, n, n)
    distribution b[j](M x) = a[i](x) with C[j] = M C[i], or a (n, n, n) scalar
    b(M x) = a(x)."""
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    X = np.stack([x.ravel(), y.ravel(), z.ravel()])
    Xn = (M @ X) % n
    b = np.empty_like(a)
    if a.ndim == 3:
        b[Xn[2], Xn[1], Xn[0]] = a[X[2], X[1], X[0]]
        return b
    perm = [int(np.flatnonzero((R.C == M @ R.C[i]).all(axis=1))[0]) for i in range(R.NVEL)]
    for i in range(R.NVEL):
        b[perm[i], Xn[2], Xn[1], Xn[0]] = a[i][X[2], X[1], X[0]]
    return b
