"""Host-side logic of the CUDA path that needs no GPU, compiled with nvcc as plain
host code: the block -> (tile, z-chunk) order of the step kernels."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")


@pytest.fixture(scope="module")
def tile_order_bin(tmp_path_factory):
    if not os.path.exists(NVCC) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    out = str(tmp_path_factory.mktemp("host") / "tile_order")
    src = os.path.join(ROOT, "tests", "host", "tile_order.cu")
    inc = os.path.join(ROOT, "paper_1609_01479_b200", "csrc")
    subprocess.run([NVCC if os.path.exists(NVCC) else "nvcc", "-std=c++17", "-I", inc, src, "-o", out], check=True)
    return out


@pytest.mark.parametrize("shape", [
    (16, 64, 2, 148),   # 512x512x64 with 32x8 tiles, two z-chunks, one CTA per SM
    (16, 64, 1, 148),
    (4, 32, 2, 296),    # 128^3 with 32x4 tiles, two CTAs per SM (one group)
    (3, 5, 4, 7),       # last group partial
    (1, 1, 3, 148),
    (16, 64, 8, 1 << 30),  # residency above the tile count: chunk-slowest order
])
def test_tile_order_is_a_bijection_with_chunks_one_group_apart(tile_order_bin, shape):
    r = subprocess.run([tile_order_bin, *map(str, shape)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout
