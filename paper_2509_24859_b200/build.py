"""Build the C-ABI library libhapt_b200.so in-tree for sm_100a.

    python -m paper_2509_24859_b200.build        (or __graft_entry__.build())

Plain nvcc, one shared object, no torch extension machinery: the library's
ABI is include/hapt_b200.h and Python reaches it through ctypes.
--fmad=false keeps every fp64 expression un-contracted (bit parity with the
CPU reference); the kernels also spell out the rounding
with __dadd_rn/__dmul_rn/__ddiv_rn.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = ["hapt_runtime.cu", "hapt_tables.cu", "hapt_dp.cu", "hapt_sim.cu", "hapt_frontend.cpp"]
LIB = os.path.join(PKG, "libhapt_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags() -> list[str]:
    return ARCH + [
        "-O3",
        "-lineinfo",
        "--fmad=false",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC,-ffp-contract=off",
        "-Xptxas",
        "-v",
        f"-I{os.path.join(REPO, 'include')}",
    ]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(REPO, "include", "hapt_b200.h"))
    deps.append(os.path.abspath(__file__))
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every source and link LIB (or `out` for an experimental variant
    built with extra -D defines, e.g. HAPT_RELAX_MINB=4)."""
    lib = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    build_dir = os.path.join(PKG, "build" if not defines else "build_variant")
    os.makedirs(build_dir, exist_ok=True)
    objs = []
    log = []
    for src in SOURCES:
        obj = os.path.join(build_dir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *flags(), *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src),
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    with open(os.path.join(build_dir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=os.path.join(PKG, outs[0]) if outs else None))
