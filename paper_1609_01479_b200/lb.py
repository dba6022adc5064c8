"""Thin ctypes binding of the C ABI in include/lb.h (argument marshalling only).

Every step of the path runs in liblb.so's CUDA kernels; this module only
converts arrays to pointers and return codes to exceptions.  There is no CPU
fallback: if liblb.so is missing or fails to load, importing this module
raises.  Function names follow the C ABI (``lb_create``, ``lb_set_state``,
``lb_step``, ``lb_get_state``, ``lb_destroy`` ...); ``Lattice`` is a small
owning wrapper around a handle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# LB_VARIANT=<name> loads liblb_<name>.so from this directory instead: the
# bounds-checked test build (checked: device index checks, lb_debug_check), or
# another build of the same sources kept for an A/B measurement; test support only
_VARIANT = os.environ.get("LB_VARIANT", "")
_LIB_NAME = f"liblb_{_VARIANT}.so" if _VARIANT else "liblb.so"
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), _LIB_NAME)
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)"
    )
_lib = C.CDLL(_LIB_PATH)

LB_OK, LB_EINVAL, LB_ENOMEM, LB_ECUDA, LB_ENCCL, LB_ESTATE, LB_ENUMERIC = 0, -1, -2, -3, -4, -5, -6
_NAMES = {-1: "LB_EINVAL", -2: "LB_ENOMEM", -3: "LB_ECUDA", -4: "LB_ENCCL", -5: "LB_ESTATE", -6: "LB_ENUMERIC"}
Q = 19


class LBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class lb_params(C.Structure):
    _fields_ = [("tau_f", C.c_double), ("tau_g", C.c_double), ("A", C.c_double), ("B", C.c_double),
                ("kappa", C.c_double), ("mobility", C.c_double)]


_vp, _dp, _i, _ll = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_longlong


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_lib_version = _sig("lb_version", C.c_char_p)
_lb_create = _sig("lb_create", _i, _i, _i, _i, C.POINTER(lb_params), C.POINTER(_vp))
_lb_create_loopback = _sig("lb_create_loopback", _i, _i, _i, _i, C.POINTER(lb_params), _i, C.POINTER(_vp))
_lb_nccl_get_unique_id = _sig("lb_nccl_get_unique_id", _i, _vp)
_lb_create_slab = _sig("lb_create_slab", _i, _i, _i, _i, C.POINTER(lb_params), _i, _i, _vp, C.POINTER(_vp))
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
_lb_create_slab_ext = _sig("lb_create_slab_ext", _i, _i, _i, _i, C.POINTER(lb_params), _i, _i, ALLGATHER_FN, _vp,
                           C.POINTER(_vp))
_lb_debug_step_phase = _sig("lb_debug_step_phase", _i, _vp, _i)
_lb_local_sites = _sig("lb_local_sites", C.c_size_t, _vp)
_lb_set_state = _sig("lb_set_state", _i, _vp, _vp, _vp)
_lb_init_equilibrium = _sig("lb_init_equilibrium", _i, _vp, _vp, _vp, _vp)
_lb_step = _sig("lb_step", _i, _vp, _i)
_lb_prepare = _sig("lb_prepare", _i, _vp)
_lb_debug_stream = _sig("lb_debug_stream", _i, _vp, _i)
_lb_debug_tune = _sig("lb_debug_tune", _i, _vp, _i, _i)
_lb_debug_step_kernel = _sig("lb_debug_step_kernel", _i, _vp, _i)
_lb_get_state = _sig("lb_get_state", _i, _vp, _vp, _vp)
_lb_get_phi = _sig("lb_get_phi", _i, _vp, _vp)
_lb_destroy = _sig("lb_destroy", None, _vp)
_lb_last_error = _sig("lb_last_error", C.c_char_p, _vp)
_lb_stream = _sig("lb_stream", _vp, _vp)
_lb_launch_count = _sig("lb_launch_count", _ll, _vp)
_lb_profile_enable = _sig("lb_profile_enable", _i, _vp, _i)
_lb_profile_reset = _sig("lb_profile_reset", _i, _vp)
_lb_profile_count = _sig("lb_profile_count", _i, _vp)
_lb_profile_entry = _sig("lb_profile_entry", _i, _vp, _i, C.POINTER(C.c_char_p), _dp, C.POINTER(_ll))
_lb_bytes_per_site = _sig("lb_bytes_per_site", C.c_double)
_lb_debug_propagation_map = _sig("lb_debug_propagation_map", _i, _i, _i, _i, _i, _vp)
_lb_debug_propagation_map_peers = _sig("lb_debug_propagation_map_peers", _i, _i, _i, _i, _i, _vp)
_lb_debug_halo_mode = _sig("lb_debug_halo_mode", _i, _vp, _i)
_lb_debug_guards = _sig("lb_debug_guards", _ll, _vp)
_lb_debug_check = _sig("lb_debug_check", _i, _vp)
_lb_debug_checked = _sig("lb_debug_checked", _i)
_lb_debug_tile_order = _sig("lb_debug_tile_order", _i, _i, _i, _i, _i, _i, _vp)
_lb_halo_plan = _sig("lb_halo_plan", _i, _i, _i, _i, _i, _i, _vp)
_lb_set_collision = _sig("lb_set_collision", _i, _vp, _i, C.c_double, C.c_double, C.c_double)
_lb_create_ch = _sig("lb_create_ch", _i, _i, _i, _i, C.POINTER(lb_params), C.c_double, C.c_double, C.c_double,
                     C.POINTER(_vp))
_lb_create_ch_loopback = _sig("lb_create_ch_loopback", _i, _i, _i, _i, C.POINTER(lb_params), C.c_double, C.c_double,
                              C.c_double, _i, C.POINTER(_vp))
_lb_create_ch_slab = _sig("lb_create_ch_slab", _i, _i, _i, _i, C.POINTER(lb_params), C.c_double, C.c_double,
                          C.c_double, _i, _i, _vp, C.POINTER(_vp))
_lb_set_state_ch = _sig("lb_set_state_ch", _i, _vp, _vp, _vp)
_lb_get_state_ch = _sig("lb_get_state_ch", _i, _vp, _vp, _vp)


class lb_lc_params(C.Structure):
    _fields_ = [("tau_f", C.c_double), ("A0", C.c_double), ("gamma", C.c_double), ("kappa", C.c_double),
                ("xi", C.c_double), ("Gamma", C.c_double)]


_lb_create_lc = _sig("lb_create_lc", _i, _i, _i, _i, C.POINTER(lb_lc_params), C.POINTER(_vp))
_lb_create_lc_loopback = _sig("lb_create_lc_loopback", _i, _i, _i, _i, C.POINTER(lb_lc_params), _i, C.POINTER(_vp))
_lb_create_lc_slab = _sig("lb_create_lc_slab", _i, _i, _i, _i, C.POINTER(lb_lc_params), _i, _i, _vp, C.POINTER(_vp))
_lb_set_state_lc = _sig("lb_set_state_lc", _i, _vp, _vp, _vp, _vp)
_lb_get_state_lc = _sig("lb_get_state_lc", _i, _vp, _vp, _vp, _vp)
_lb_init_lc = _sig("lb_init_lc", _i, _vp, _vp, _vp, _vp)

EXPORTS = [
    "lb_version", "lb_create", "lb_create_loopback", "lb_nccl_get_unique_id", "lb_create_slab", "lb_create_slab_ext", "lb_debug_step_phase", "lb_local_sites",
    "lb_set_state", "lb_init_equilibrium", "lb_step", "lb_prepare", "lb_debug_stream", "lb_debug_tune", "lb_debug_step_kernel", "lb_get_state", "lb_get_phi", "lb_destroy",
    "lb_last_error", "lb_stream", "lb_launch_count", "lb_profile_enable", "lb_profile_reset", "lb_profile_count",
    "lb_profile_entry", "lb_bytes_per_site", "lb_debug_propagation_map", "lb_debug_propagation_map_peers",
    "lb_debug_halo_mode", "lb_debug_tile_order", "lb_debug_guards", "lb_debug_check", "lb_debug_checked", "lb_halo_plan", "lb_set_collision", "lb_create_ch", "lb_create_ch_loopback", "lb_create_ch_slab", "lb_set_state_ch",
    "lb_get_state_ch",
    "lb_create_lc", "lb_create_lc_loopback", "lb_create_lc_slab", "lb_set_state_lc", "lb_get_state_lc", "lb_init_lc",
]


def _check(rc: int, h) -> None:
    if rc != LB_OK:
        raise LBError(rc, (_lb_last_error(h) or b"").decode())


def _ptr(a, n: int, writable: bool = False) -> int:
    """Pointer to n contiguous float64 values: a NumPy array or a (CPU, possibly
    pinned) torch tensor.  No copies: a non-conforming array raises."""
    if hasattr(a, "data_ptr"):  # torch tensor
        if a.device.type != "cpu" or a.dtype.__repr__() != "torch.float64" or not a.is_contiguous() or a.numel() != n:
            raise ValueError(f"need a contiguous CPU float64 tensor of {n} elements")
        return a.data_ptr()
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or a.size != n:
        raise ValueError(f"need a C-contiguous float64 ndarray of {n} elements")
    if writable and not a.flags.writeable:
        raise ValueError("output array is read-only")
    return a.ctypes.data


def make_params(tau_f=0.8, tau_g=1.3, A=-0.0625, B=0.0625, kappa=0.04, mobility=0.05) -> lb_params:
    return lb_params(tau_f, tau_g, A, B, kappa, mobility)


# ---- C ABI names ------------------------------------------------------------
def lb_version() -> str:
    return _lib_version().decode()


def lb_create(nx: int, ny: int, nz: int, params: lb_params):
    h = _vp()
    _check(_lb_create(nx, ny, nz, C.byref(params), C.byref(h)), None)
    return h


def lb_create_loopback(nx: int, ny: int, nz: int, params: lb_params, nslabs: int):
    h = _vp()
    _check(_lb_create_loopback(nx, ny, nz, C.byref(params), nslabs, C.byref(h)), None)
    return h


def lb_nccl_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lb_nccl_get_unique_id(buf), None)
    return buf.raw


def lb_create_slab(nx: int, ny: int, nz: int, params: lb_params, nranks: int, rank: int, uid: bytes | None):
    h = _vp()
    buf = C.create_string_buffer(uid, 128) if uid is not None else None
    _check(_lb_create_slab(nx, ny, nz, C.byref(params), nranks, rank, buf, C.byref(h)), None)
    return h


def lb_create_slab_ext(nx: int, ny: int, nz: int, params: lb_params, nranks: int, rank: int, allgather):
    """lb_create_slab bootstrapped by `allgather(mine: bytes) -> bytes` (nranks * len(mine),
    rank order; e.g. dist.allgather_bytes).  Returns (handle, callback); keep the
    callback alive as long as the handle (the library calls it until lb_destroy)."""

    def cb(_ctx, send, recv, nbytes):
        try:
            out = allgather(C.string_at(send, nbytes))
            if len(out) != nranks * nbytes:
                return -1
            C.memmove(recv, out, len(out))
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed all-gather
            return -1

    fn = ALLGATHER_FN(cb)
    h = _vp()
    _check(_lb_create_slab_ext(nx, ny, nz, C.byref(params), nranks, rank, fn, None, C.byref(h)), None)
    return h, fn


def lb_debug_step_phase(h, phase: int) -> None:
    _check(_lb_debug_step_phase(h, phase), h)


def lb_local_sites(h) -> int:
    return int(_lb_local_sites(h))


def lb_set_state(h, f, g) -> None:
    n = Q * lb_local_sites(h)
    _check(_lb_set_state(h, _ptr(f, n), _ptr(g, n)), h)


def lb_init_equilibrium(h, rho, u, phi) -> None:
    n = lb_local_sites(h)
    _check(_lb_init_equilibrium(h, None if rho is None else _ptr(rho, n), None if u is None else _ptr(u, 3 * n),
                                _ptr(phi, n)), h)


def lb_step(h, nsteps: int) -> None:
    _check(_lb_step(h, nsteps), h)


def lb_prepare(h) -> None:
    _check(_lb_prepare(h), h)


def lb_debug_stream(h, nsteps: int) -> None:
    _check(_lb_debug_stream(h, nsteps), h)


def lb_debug_step_kernel(h, which: int) -> None:
    _check(_lb_debug_step_kernel(h, which), h)


# lb_debug_tune keys (include/lb.h)
LB_TUNE_ZCHUNK, LB_TUNE_BAND_ROWS, LB_TUNE_RESID, LB_TUNE_GRAPHS = 1, 2, 3, 4
LB_TUNE_L2_BOX, LB_TUNE_L2_FTILE, LB_TUNE_L2_GTILE, LB_TUNE_TILE_ROWS, LB_TUNE_VARIANT = 5, 6, 7, 8, 9


def lb_debug_tune(h, key: int, value: int) -> None:
    _check(_lb_debug_tune(h, key, value), h)


def lb_get_state(h, f=None, g=None):
    n = Q * lb_local_sites(h)
    f = np.empty(n) if f is None else f
    g = np.empty(n) if g is None else g
    _check(_lb_get_state(h, _ptr(f, n, True), _ptr(g, n, True)), h)
    return f, g


def lb_get_phi(h, phi=None):
    n = lb_local_sites(h)
    phi = np.empty(n) if phi is None else phi
    _check(_lb_get_phi(h, _ptr(phi, n, True)), h)
    return phi


def lb_destroy(h) -> None:
    _lb_destroy(h)


def lb_last_error(h=None) -> str:
    return (_lb_last_error(h) or b"").decode()


def lb_stream(h) -> int:
    return int(_lb_stream(h) or 0)


def lb_launch_count(h) -> int:
    return int(_lb_launch_count(h))


def lb_profile_enable(h, on: bool) -> None:
    _check(_lb_profile_enable(h, int(on)), h)


def lb_profile_reset(h) -> None:
    _check(_lb_profile_reset(h), h)


def lb_profile(h) -> dict:
    """{kernel name: (total device ms, timed launches)} from the handle's event timers."""
    out = {}
    for i in range(_lb_profile_count(h)):
        name, ms, n = C.c_char_p(), C.c_double(), _ll()
        _check(_lb_profile_entry(h, i, C.byref(name), C.byref(ms), C.byref(n)), h)
        out[name.value.decode()] = (ms.value, n.value)
    return out


def lb_bytes_per_site() -> float:
    return float(_lb_bytes_per_site())


def lb_debug_propagation_map(nx: int, ny: int, nz: int, nslabs: int = 1) -> np.ndarray:
    out = np.empty(Q * nx * ny * nz, dtype=np.int64)
    rc = _lb_debug_propagation_map(nx, ny, nz, nslabs, out.ctypes.data)
    if rc != LB_OK:
        raise LBError(rc, "propagation map failed (bad sizes or not a permutation)")
    return out.reshape(Q, nz, ny, nx)


def lb_debug_propagation_map_peers(nx: int, ny: int, nz: int, nslabs: int = 1) -> np.ndarray:
    out = np.empty(Q * nx * ny * nz, dtype=np.int64)
    rc = _lb_debug_propagation_map_peers(nx, ny, nz, nslabs, out.ctypes.data)
    if rc != LB_OK:
        raise LBError(rc, "peer propagation map failed (bad sizes, a ghost-plane store or not a permutation)")
    return out.reshape(Q, nz, ny, nx)


def lb_debug_guards(h) -> int:
    """Guard-zone bytes no longer holding their pattern (0 = no store left its buffer)."""
    n = int(_lb_debug_guards(h))
    if n < 0:
        raise LBError(n, lb_last_error(h))
    return n


def lb_debug_check(h) -> int:
    """LB_CHECKED builds: source line of the first failed device bounds check (0: none)."""
    n = int(_lb_debug_check(h))
    if n < 0:
        raise LBError(n, lb_last_error(h))
    return n


def lb_debug_checked() -> bool:
    return bool(_lb_debug_checked())


def lb_debug_tile_order(ntx: int, nty: int, nch: int, resid: int, band: int = 1) -> np.ndarray:
    out = np.empty((ntx * nty * nch, 3), dtype=np.int32)
    rc = _lb_debug_tile_order(ntx, nty, nch, resid, band, out.ctypes.data)
    if rc != LB_OK:
        raise LBError(rc, "lb_debug_tile_order: bad arguments")
    return out


def lb_set_collision(h, model: int, tau_shear: float = 0.8, tau_bulk: float = 1.0, tau_ghost: float = 1.0) -> None:
    """0: BGK + Guo force (default); 1: chemical stress in f^eq with a three-rate MRT."""
    _check(_lb_set_collision(h, model, tau_shear, tau_bulk, tau_ghost), h)


def lb_create_ch(nx: int, ny: int, nz: int, params: lb_params, tau_shear=0.8, tau_bulk=1.1, tau_ghost=1.0):
    h = _vp()
    _check(_lb_create_ch(nx, ny, nz, C.byref(params), tau_shear, tau_bulk, tau_ghost, C.byref(h)), None)
    return h.value


def lb_create_ch_loopback(nx: int, ny: int, nz: int, params: lb_params, tau_shear, tau_bulk, tau_ghost, nslabs: int):
    h = _vp()
    _check(_lb_create_ch_loopback(nx, ny, nz, C.byref(params), tau_shear, tau_bulk, tau_ghost, nslabs, C.byref(h)),
           None)
    return h.value


def lb_create_ch_slab(nx: int, ny: int, nz: int, params: lb_params, tau_shear, tau_bulk, tau_ghost, nranks: int,
                      rank: int, uid: bytes):
    h = _vp()
    buf = C.create_string_buffer(uid, 128)
    _check(_lb_create_ch_slab(nx, ny, nz, C.byref(params), tau_shear, tau_bulk, tau_ghost, nranks, rank, buf,
                              C.byref(h)), None)
    return h.value


def lb_set_state_ch(h, f, phi) -> None:
    n = lb_local_sites(h)
    _check(_lb_set_state_ch(h, _ptr(f, Q * n), _ptr(phi, n)), h)


def lb_get_state_ch(h, f=None, phi=None):
    n = lb_local_sites(h)
    f = np.empty(Q * n) if f is None else f
    phi = np.empty(n) if phi is None else phi
    _check(_lb_get_state_ch(h, _ptr(f, Q * n, True), _ptr(phi, n, True)), h)
    return f, phi


def make_lc_params(tau_f=0.8, A0=0.01, gamma=3.2, kappa=0.01, xi=0.7, Gamma=0.3) -> lb_lc_params:
    """Defaults: DESIGN.md R44."""
    return lb_lc_params(tau_f, A0, gamma, kappa, xi, Gamma)


def lb_create_lc(nx: int, ny: int, nz: int, params: lb_lc_params):
    h = _vp()
    _check(_lb_create_lc(nx, ny, nz, C.byref(params), C.byref(h)), None)
    return h.value


def lb_create_lc_loopback(nx: int, ny: int, nz: int, params: lb_lc_params, nslabs: int):
    h = _vp()
    _check(_lb_create_lc_loopback(nx, ny, nz, C.byref(params), nslabs, C.byref(h)), None)
    return h.value


def lb_create_lc_slab(nx: int, ny: int, nz: int, params: lb_lc_params, nranks: int, rank: int, uid: bytes):
    h = _vp()
    buf = C.create_string_buffer(uid, 128)
    _check(_lb_create_lc_slab(nx, ny, nz, C.byref(params), nranks, rank, buf, C.byref(h)), None)
    return h.value


def lb_set_state_lc(h, f, q, u) -> None:
    n = lb_local_sites(h)
    _check(_lb_set_state_lc(h, _ptr(f, Q * n), _ptr(q, 5 * n), _ptr(u, 3 * n)), h)


def lb_get_state_lc(h, f=None, q=None, u=None):
    n = lb_local_sites(h)
    f = np.empty(Q * n) if f is None else f
    q = np.empty(5 * n) if q is None else q
    u = np.empty(3 * n) if u is None else u
    _check(_lb_get_state_lc(h, _ptr(f, Q * n, True), _ptr(q, 5 * n, True), _ptr(u, 3 * n, True)), h)
    return f, q, u


def lb_init_lc(h, rho, u, n_dir) -> None:
    n = lb_local_sites(h)
    _check(_lb_init_lc(h, None if rho is None else _ptr(rho, n), None if u is None else _ptr(u, 3 * n),
                       _ptr(n_dir, 3 * n)), h)


def lb_debug_halo_mode(h, mode: int = -1) -> int:
    """-1: query (returns 0 exchange / 1 peer); 0 or 1: set (returns 0)."""
    rc = _lb_debug_halo_mode(h, mode)
    if rc < 0:
        _check(rc, h)
    return rc


def lb_halo_plan(nx: int, ny: int, nz: int, nranks: int, rank: int) -> dict:
    out = np.empty(4, dtype=np.int64)
    _check(_lb_halo_plan(nx, ny, nz, nranks, rank, out.ctypes.data), None)
    return {"up": int(out[0]), "down": int(out[1]), "dist_doubles": int(out[2]), "phi_doubles": int(out[3])}


# ---- owning wrapper -----------------------------------------------------------
class Lattice:
    """A handle plus its shape.  Arrays at this level are (19, nz, ny, nx)."""

    def __init__(self, nx, ny, nz, params: lb_params | None = None, nslabs: int = 1, nranks: int = 1, rank: int = 0,
                 uid: bytes | None = None, allgather=None):
        """nranks > 1: one rank of a z-slab decomposition, bootstrapped by NCCL (uid from
        lb_nccl_get_unique_id) or, with `allgather` (bytes -> bytes), by the caller."""
        self.params = params or make_params()
        self._cb = None
        if nranks > 1 and allgather is not None:
            self.h, self._cb = lb_create_slab_ext(nx, ny, nz, self.params, nranks, rank, allgather)
            self.shape = (nz // nranks, ny, nx)
        elif nranks > 1:
            self.h = lb_create_slab(nx, ny, nz, self.params, nranks, rank, uid)
            self.shape = (nz // nranks, ny, nx)
        else:
            self.h = lb_create_loopback(nx, ny, nz, self.params, nslabs) if nslabs > 1 else lb_create(nx, ny, nz, self.params)
            self.shape = (nz, ny, nx)

    def close(self):
        h = getattr(self, "h", None)
        if h:
            lb_destroy(h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_state(self, f, g):
        lb_set_state(self.h, np.ascontiguousarray(f, dtype=np.float64).reshape(-1),
                     np.ascontiguousarray(g, dtype=np.float64).reshape(-1))

    def init_equilibrium(self, phi, rho=None, u=None):
        c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        lb_init_equilibrium(self.h, c(rho), c(u), c(phi))

    def step(self, n: int = 1):
        lb_step(self.h, n)

    def stream_only(self, n: int = 1):
        lb_debug_stream(self.h, n)

    def get_state(self):
        f, g = lb_get_state(self.h)
        return f.reshape((Q,) + self.shape), g.reshape((Q,) + self.shape)

    def get_phi(self):
        return lb_get_phi(self.h).reshape(self.shape)


class ChLattice(Lattice):
    """A finite-difference Cahn-Hilliard handle (lb_create_ch): state (f, phi)."""

    def __init__(self, nx, ny, nz, params: lb_params | None = None, tau_shear=0.8, tau_bulk=1.1, tau_ghost=1.0,
                 nslabs: int = 1, nranks: int = 1, rank: int = 0, uid: bytes | None = None):
        self.params = params or make_params()
        t = (tau_shear, tau_bulk, tau_ghost)
        if nranks > 1:
            self.h = lb_create_ch_slab(nx, ny, nz, self.params, *t, nranks, rank, uid)
            self.shape = (nz // nranks, ny, nx)
        else:
            self.h = (lb_create_ch_loopback(nx, ny, nz, self.params, *t, nslabs) if nslabs > 1
                      else lb_create_ch(nx, ny, nz, self.params, *t))
            self.shape = (nz, ny, nx)

    def set_state(self, f, phi):
        lb_set_state_ch(self.h, np.ascontiguousarray(f, dtype=np.float64).reshape(-1),
                        np.ascontiguousarray(phi, dtype=np.float64).reshape(-1))

    def get_state(self):
        f, phi = lb_get_state_ch(self.h)
        return f.reshape((Q,) + self.shape), phi.reshape(self.shape)


class LcLattice(Lattice):
    """A liquid-crystal handle (lb_create_lc, NEXT-4): state (f, Q, u); arrays are
    (19 | 5 | 3, nz, ny, nx)."""

    def __init__(self, nx, ny, nz, params: lb_lc_params | None = None, nslabs: int = 1, nranks: int = 1,
                 rank: int = 0, uid: bytes | None = None):
        self.params = params or make_lc_params()
        if nranks > 1:
            self.h = lb_create_lc_slab(nx, ny, nz, self.params, nranks, rank, uid)
            self.shape = (nz // nranks, ny, nx)
        else:
            self.h = (lb_create_lc_loopback(nx, ny, nz, self.params, nslabs) if nslabs > 1
                      else lb_create_lc(nx, ny, nz, self.params))
            self.shape = (nz, ny, nx)

    def set_state(self, f, q, u):
        c = lambda a: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)  # noqa: E731
        lb_set_state_lc(self.h, c(f), c(q), c(u))

    def init(self, n_dir, rho=None, u=None):
        c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(-1)  # noqa: E731
        lb_init_lc(self.h, c(rho), c(u), c(n_dir))

    def get_state(self):
        f, q, u = lb_get_state_lc(self.h)
        return f.reshape((Q,) + self.shape), q.reshape((5,) + self.shape), u.reshape((3,) + self.shape)
