"""In-tree build of libmbci.so (nvcc, sm_100a).  The .so lands next to this file so it
travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmbci.so")
LIB_TRACE = os.path.join(HERE, "libmbci_trace.so")
# api.cu (ABI + host logic), selector.cpp, and one translation unit per kernel family / dtype
# (k_*.cu), compiled in parallel and linked into one shared library.
SOURCES = [os.path.join(CSRC, f) for f in ("api.cu", "selector.cpp", "search.cpp", "prune.cpp")] + sorted(
    os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.startswith("k_") and f.endswith(".cu"))
DEPS = SOURCES + [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cuh", ".h"))] + [
    os.path.join(os.path.dirname(HERE), "include", "mbci.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def stale_lib(lib) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines=()) -> str:
    """libmbci.so (production) or, with trace=True, libmbci_trace.so (per-CTA event timestamps
    compiled in; loaded by the binding when MBCI_LIB=trace — diagnostics only).  variant + defines:
    an A/B copy libmbci_<variant>.so compiled with -D<defines> (MBCI_LIB=ab:libmbci_<variant>.so)."""
    lib = LIB_TRACE if trace else (os.path.join(HERE, f"libmbci_{variant}.so") if variant else LIB)
    if force or stale_lib(lib):
        extra = (["-DMBCI_TRACE=1"] if trace else []) + [f"-D{d}" for d in defines]
        # objects outside the repo: only the linked .so travels to the GPU box
        objdir = os.path.join(tempfile.gettempdir(), "mbci_build",
                              "trace" if trace else (variant or "release"))
        os.makedirs(objdir, exist_ok=True)
        objs, procs = [], []
        for src in SOURCES:
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            objs.append(obj)
            cmd = [nvcc()] + NVCC_FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
            procs.append((src, subprocess.Popen(cmd)))
        failed = [src for src, pr in procs if pr.wait() != 0]
        if failed:
            raise RuntimeError("nvcc failed for " + ", ".join(os.path.basename(f) for f in failed))
        subprocess.check_call([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib + ".tmp"]
                              + objs)
        os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
