"""Build libquartet_b200.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_2505_14669_b200.build          # or __graft_entry__.build()
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(BUILD, "libquartet_b200.so")
SOURCES = ["quant.cu", "tcq.cu", "tcq_x.cu", "gemm.cu", "glue.cu", "seam.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "quartet_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """Compile the sources in parallel and link LIB.  `defines` / `out`: an experiment build (e.g.
    ("QT_WAIT_HINT=1",) into another directory, loaded with QT_LIB_PATH); production uses neither."""
    lib = LIB if out is None else os.path.join(out, "libquartet_b200.so")
    if out is None and not force and not _stale():
        return LIB
    bdir = os.path.dirname(lib)
    os.makedirs(bdir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed ({p.args[-3]})")
    LIB_ = lib
    tmp = LIB_ + ".tmp"
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link of {LIB_} failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB_)
    return LIB_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
