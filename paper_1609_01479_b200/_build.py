"""Build liblb.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblb.so")
LIB_CHECKED = os.path.join(PKG, "liblb_checked.so")  # -DLB_CHECKED: device bounds checks (test support)
SOURCES = ["lb_kernels.cu", "lb_step.cu", "lb_step_ws.cu", "lb_step_ch.cu", "lb_step_lc.cu", "lb_api.cu"]
HEADERS = ["d3q19.cuh", "lb_kernels.cuh", "lb_device.cuh", "lb_tma.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    """NCCL headers/library of the torch-bundled nvidia-nccl wheel (2.28), so the
    process loads one libnccl.so.2 whether torch or liblb loads it first."""
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "lb.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile every source to an object in parallel, then link liblb.so (checked:
    liblb_checked.so, the same sources with -DLB_CHECKED)."""
    out = LIB_CHECKED if checked else LIB
    if not force and not _stale(out):
        return out
    inc, lib = nccl_dirs()
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
             "-Xptxas", "-v" if verbose else "-O3",
             "-I", os.path.join(ROOT, "include"), "-I", inc,
             *(["-DLB_CHECKED"] if checked else []),
             *os.environ.get("LB_NVCC_FLAGS", "").split()]
    objdir = os.path.join(PKG, "build_obj_checked" if checked else "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.splitext(s)[0] + ".o") for s in SOURCES]

    def compile_one(src_obj):
        src, obj = src_obj
        return subprocess.run([nvcc, *flags, "-c", os.path.join(CSRC, src), "-o", obj], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, zip(SOURCES, objs)))
    for r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building liblb.so")
        if verbose:
            sys.stderr.write(r.stderr)
    r = subprocess.run([nvcc, *ARCH, "-shared", *objs, "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}",
                        "-o", out + ".tmp"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking liblb.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
