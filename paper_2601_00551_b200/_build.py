"""Build the sm_100a shared library in-tree (no JIT cache, travels with the
repo snapshot): ``paper_2601_00551_b200/libpaball_b200.so``."""

from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpaball_b200.so")
SOURCES = ["pab_pack.cu", "pab_sort.cu", "pab_forward.cu", "pab_adjoint.cu", "pab_driver.cu", "pab_density.cu", "pab_render.cu",
           "pab_ubp.cu", "pab_host.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "paball_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines: tuple = ()) -> str:
    """Compile every source into one shared library (``defines``: extra -D
    tuning macros for experiment builds written to ``out``)."""
    if out == LIB and not force and not needs_build():
        return LIB
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", *[f"-D{d}" for d in defines]]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    os.replace(out + ".tmp", out)
    if verbose:
        print(res.stdout + res.stderr)
    return out


def build_probe() -> str:
    """FP32/ex2 peak probe used by bench.py for the roofline denominator
    (measurement tooling, not part of the product library)."""
    src = os.path.join(ROOT, "tools", "probe", "fp32_peak.cu")
    out = os.path.join(ROOT, "tools", "probe", "libfp32_peak.so")
    cmd = [nvcc(), *ARCH, "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", out, src]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed (probe):\n" + res.stdout + res.stderr)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
