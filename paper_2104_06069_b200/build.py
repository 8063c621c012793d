"""Build the in-tree sm_100a shared library libbitlamb_b200.so.

nvcc cross-compiles for sm_100a without a GPU.  The kernels are compiled with
-fmad=false (the reference's x86-64 arithmetic has no FMA contraction) and
-lineinfo (ncu source view).  NCCL is the torch-bundled libnccl.so.2, the one
a `torch.distributed` process has already loaded.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbitlamb_b200.so")
SOURCES = ["bl_kernels.cu", "bl_runtime.cu"]
HEADERS = ["bl_kernels.cuh", "bl_runtime.h", os.path.join("..", "..", "include", "bitlamb_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("NCCL headers/library not found")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Build the library; `out`/`defines` make A/B variants (-D tuning knobs)."""
    if out == OUT and not defines and not force and not needs_build():
        return OUT
    inc, lib = nccl_dirs()
    host_cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-ccbin", host_cxx,
           "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared", f"-I{inc}",
           *[os.path.join(CSRC, s) for s in SOURCES],
           f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}", "-lcudart",
           *defines, "-o", out + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DKNOB=V ...]  (variants for A/B timing)
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else OUT
    defs = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=os.path.abspath(out), defines=defs))
