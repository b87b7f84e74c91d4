"""Build the in-tree C-ABI library `_dz_b200.so` with nvcc for sm_100a (no torch involved)."""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_dz_b200.so")
BUILD = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}"]

SOURCES = ["dz_codec.cu", "dz_sbmm.cu", "dz_prefill.cu", "dz_tp.cu", "dz_plan.cu", "dz_sched.cu", "dz_obs.cu",
           "dz_host.cpp", "dz_dzdl.cpp"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False, variant: str = "",
          defines: list[str] | None = None) -> str:
    """Build `_dz_b200.so`, the DZ_TRACE-instrumented `_dz_b200_trace.so` (tools/trace.py), or an
    experiment variant `_dz_b200_<variant>.so` with extra -D defines (loaded via DZ_B200_LIB)."""
    global LIB, BUILD
    defines = list(defines or [])
    if trace:
        variant, defines = "trace", defines + ["-DDZ_TRACE"]
    if variant:
        LIB = os.path.join(PKG, f"_dz_b200_{variant}.so")
        BUILD = os.path.join(ROOT, "build", f"obj_{variant}")
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "dz_b200.h"))
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [NVCC, *ARCH, *NVFLAGS, *defines, "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lz"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    print(build(verbose=True, force="--force" in sys.argv, trace="--trace" in sys.argv, variant=var,
                defines=[a for a in sys.argv[1:] if a.startswith("-D")]))
