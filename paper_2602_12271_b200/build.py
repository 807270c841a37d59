"""Build the in-tree C-ABI library ``libmonarch_b200.so`` for sm_100a.

    python -m paper_2602_12271_b200.build          # or __graft_entry__.build()

nvcc cross-compiles without a GPU; the resulting .so sits next to this file
and travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmonarch_b200.so")
SOURCES = ("mbx_api.cu", "mbx_generic.cu", "mbx_tc.cu", "mbx_backward.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "monarch_b200.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """trace=True builds libmonarch_b200_trace.so with per-CTA event timestamps
    (MBX_TRACE; a profiling aid, never loaded unless MBX_LIB points at it).
    ``variant`` + ``defines`` build libmonarch_b200_<variant>.so with extra -D flags
    (A/B experiments, loaded through MBX_LIB only)."""
    lib = LIB.replace(".so", "_trace.so") if trace else LIB
    if variant:
        lib = LIB.replace(".so", f"_{variant}.so")
    if not force and not trace and not variant and not _stale():
        return LIB
    objs = []
    tmp = os.path.join(HERE, "_build")
    os.makedirs(tmp, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-diag-suppress", "177", "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags += ["-Xptxas", "-v"]
    if trace:
        flags += ["-DMBX_TRACE"]
    flags += [f"-D{d}" for d in defines]
    suffix = ("_trace" if trace else "") + (f"_{variant}" if variant else "")
    for src in SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", suffix + ".o"))
        cmd = [nvcc(), "-c", os.path.join(CSRC, src), "-o", obj] + flags
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp_lib = lib + ".tmp"
    subprocess.run([nvcc(), "-shared", "-o", tmp_lib] + objs + ARCH + ["-lcuda", "-ldl"], check=True)
    os.replace(tmp_lib, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    defs = tuple(a[2:] for a in sys.argv if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv, variant=var,
                defines=defs))
