"""Test helper: evaluate a whole-lattice oracle step only at sampled sites, on a
periodic window of radius r around each site (the step is local: every output of
the binary-fluid, MRT and Cahn-Hilliard steps depends on inputs within radius 3),
keeping the centre.  For parity at the bench's full sizes, where the oracle cannot
step the whole lattice in seconds."""
import numpy as np


def window(a: np.ndarray, x: int, y: int, z: int, r: int) -> np.ndarray:
    """Periodic window of radius r around (x, y, z) of a (..., nz, ny, nx) array."""
    nz, ny, nx = a.shape[-3:]
    zi = np.arange(z - r, z + r + 1) % nz
    yi = np.arange(y - r, y + r + 1) % ny
    xi = np.arange(x - r, x + r + 1) % nx
    return a[..., zi[:, None, None], yi[None, :, None], xi[None, None, :]]


def crop(a: np.ndarray, k: int = 1) -> np.ndarray:
    """Drop k layers on every side of the last three axes."""
    return a[..., k:-k, k:-k, k:-k]


def centre(a: np.ndarray) -> np.ndarray:
    r = a.shape[-1] // 2
    return a[..., r, r, r]
