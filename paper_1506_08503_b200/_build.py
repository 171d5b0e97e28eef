"""Build libgaes_b200.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

The shared library is the product: CUDA kernels (csrc/kernels.cu) plus the
C-ABI host runtime (csrc/abi.cpp, host_pipeline.cpp, device_ctx.cpp,
runtime.cpp), statically linked against cudart
so it loads without torch and ships to the GPU box inside the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "libgaes_b200.so")
SOURCES = ["kernels.cu", "runtime.cpp", "device_ctx.cpp", "host_pipeline.cpp", "abi.cpp"]
HEADERS = ["gf.cuh", "aes_ttable.cuh", "aes_bitslice.cuh", "kernels.h", "types.h", "host_pool.h", "round_keys.h",
           "runtime.h", "device_ctx.h", "host_pipeline.h", "tma.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
                     "-Xptxas", "-O3", "-I", os.path.join(REPO, "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(REPO, "include", "gaes_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def is_stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(f) > t for f in _inputs() if os.path.exists(f))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale():
        build_pyfast()
        return LIB_PATH
    nvcc = _nvcc()
    objdir = os.path.join(PKG_DIR, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB_PATH + ".tmp"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"])
    os.replace(tmp, LIB_PATH)
    build_pyfast(force=True)
    return LIB_PATH


def build_pyfast(force: bool = False) -> str:
    """csrc/pyfast.c -> _pyfast<EXT_SUFFIX>: the CPython fast path of the
    drop-in calls (argument checks + C-ABI call without Python-level
    pointer extraction), linked against libgaes_b200.so."""
    import sysconfig
    out = os.path.join(PKG_DIR, "_pyfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    src = os.path.join(CSRC, "pyfast.c")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src),
                                                                          os.path.getmtime(LIB_PATH)):
        return out
    tmp = out + ".tmp"
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-fvisibility=hidden", "-I", sysconfig.get_paths()["include"],
                           "-I", os.path.join(REPO, "include"), src, "-o", tmp, "-L", PKG_DIR, "-l:libgaes_b200.so",
                           "-Wl,-rpath,$ORIGIN"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
