"""Memory safety of the CUDA path without compute-sanitizer (closed on this pool):
guard zones around every field buffer (lb_debug_guards) and, in the
bounds-checked build liblb_checked.so (LB_VARIANT=checked), device-side checks of
the kernels' computed indices (lb_debug_check).  scripts/sanitize_cases.py runs
every step kernel on small cases (wrapped halo boxes, one tile, slabs with both
halo transports, MRT, Cahn-Hilliard, liquid crystal) against the oracle."""
import os
import subprocess
import sys

import pytest

from paper_1609_01479_b200 import lb, _build

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant", ["", "checked"])
def test_sanitize_cases(variant):
    if variant == "checked":
        _build.build(checked=True)
    env = dict(os.environ, LB_VARIANT=variant)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all ok" in r.stdout
    assert f"bounds-checked build: {variant == 'checked'}" in r.stdout


def test_guards_after_bench_sized_step():
    """The bench lattice (512 x 512 x 64, 32 x 8 tiles, two z-chunks): guards intact."""
    from paper_1609_01479_b200 import synth

    with lb.Lattice(512, 512, 64) as L:
        L.init_equilibrium(synth.spinodal_phi(512, 512, 64, seed=0))
        L.step(3)
        assert lb.lb_debug_guards(L.h) == 0
        assert lb.lb_debug_check(L.h) == 0
