"""Build libvmi.so in-tree for sm_100a (nvcc + g++), no torch JIT.

The shared library lands in paper_1709_06948_b200/_native/ so it travels with
the repo snapshot to the GPU box.  Host pose->matrix code (pose_host.cpp) is
compiled by g++ with -ffp-contract=off (bit-exact euler_to_transform).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_native")
BUILD_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libvmi.so")

CU_SOURCES = ["k_fast.cu", "k_exact.cu", "vmi_api.cu"]
CPP_SOURCES = ["pose_host.cpp", "nm_lockstep.cpp"]
HEADERS = ["vmi_device.cuh", "vmi_types.h", "vmi_kernels.h", "nm_lockstep.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v", "-Werror", "all-warnings",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, out_dir: str | None = None,
          defines: tuple = ()) -> str:
    """Build libvmi.so; ``out_dir``/``defines`` produce variant builds for A/B runs."""
    global BUILD_DIR, LIB
    if out_dir:
        BUILD_DIR = os.path.join(out_dir, "obj")
        LIB = os.path.join(out_dir, "libvmi.so")
    os.makedirs(BUILD_DIR, exist_ok=True)
    nvcc = _nvcc()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    hdrs.append(os.path.join(HERE, "..", "include", "vmi.h"))
    objs = []
    ptxas_log = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD_DIR, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            ptxas_log.append(r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD_DIR, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = ["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
                   "-Wall", "-Werror", "-c", s, "-o", o]
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
               "-lpthread"]
        subprocess.run(cmd, check=True)
    if verbose:
        sys.stdout.write("".join(ptxas_log))
    return LIB


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    out = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")), None)
    print(build(verbose=True, force="--force" in sys.argv, out_dir=out, defines=defs))
